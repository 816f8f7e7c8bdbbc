#!/usr/bin/env python3
"""bench.py -- space-time unknowns solved per second (M*N/s, fp64) for the fast
BLTT solver, BASELINE.json config 4 (time-fractional diffusion, gamma 0.3,
M = 65536 interior nodes, N = 65536 steps) by default.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one ft_solve_fast over the device-resident right-hand side
(34.4 GB in, 34.4 GB out; inputs far larger than the 126 MB L2, so no flush
is needed).  `e2e` runs the same solve through the C ABI with pinned HOST
buffers (H2D of the RHS and D2H of the solution inside the timed region).
`--impl reference` times the unmodified reference CPU solver (oracle/_ref,
built from /root/reference by oracle/build_ref.sh) on the same workload: its
direct march (the only reference path that runs at these sizes) on M' nodes at
the full N, scaled linearly to the full M (see reference_estimate); both arms
print BASELINE.json's metric string.  Without --no-configs the line also carries
per-config sub-results for BASELINE configs 1, 2, 3 and 5 (ours and the
reference's, measured the same way).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def _metric() -> str:
    """BASELINE.json's metric string, printed identically by both arms."""
    p = ROOT / "BASELINE.json"
    try:
        return json.loads(p.read_text())["metric"]
    except Exception:  # noqa: BLE001
        return "space-time unknowns solved/sec (M\u00b7N/s, fp64) and % of HBM roofline at 1/2/4/8 B200"


METRIC = _metric()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


# DRAM bytes / algorithmic bytes of the history-product launches of one config-4
# solve, per kernel family, measured with ncu over every launch of the solve
# (profiles/ncu_r02/fp64_dram_per_launch_cfg4.csv.gz, summarised in DESIGN.md §4):
# direct n <= 128: 0.68, single-CTA FFT 256 <= n <= 4096: 0.92, 2-/4-CTA clusters
# (n = 8192, 16384): 1.00, persistent split levels (n >= 32768, their scratch ring
# partly spilling to DRAM; dead ring lines discarded from L2): 1.29 (n = 65536: 1.49,
# n = 32768: 1.09; round 1's batched launches: 2.71).
NCU_DRAM_OVER_ALG = {"direct": 0.68, "single": 0.92, "cluster": 1.00, "split": 1.29}


def mp_family(n: int) -> str:
    return "direct" if n <= 128 else "single" if n <= 4096 else "cluster" if n <= 16384 else "split"


def bytes_per_unknown(N: int) -> float:
    """B_alg = 8 B M N (1.5 D + 2), D = log2(N/64)."""
    D = max(0.0, math.log2(N / 64))
    return 8.0 * (1.5 * D + 2.0)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()  # sampler live before the timed region starts
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl" if os.environ.get("FT_BACKEND", "nccl") == "nccl" else "gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(world, value: float) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---- CPU reference arm / cpu_baseline -----------------------------------------
#
# The reference solves one problem on one thread (SPEC.md: single-threaded per
# solve; its thread pool only runs independent ladder rows), and its fast path
# (GMRES) is infeasible or fails on configs 2-5.  Its direct march
# costs O(M N^2): every node sums its whole history at every step, the same work
# per node.  A sample of M' nodes at the FULL N therefore measures the per-node
# cost in the regime of the real solve (long history rows), and the full-size
# time is that sample times M / M' (linear in M: exact in work; the sample's rows
# are cache-resident, so if anything this flatters the reference).  The raw rate
# of a full-M time prefix (N' = 128, short rows) is reported beside it.

REF_SAMPLE_NODES = {4: 2, 2: 4, 3: 2, 5: 4}   # M' of the per-config reduced-M full-N sample


def _ref_one(w, method="direct"):
    """One reference solve through its public API (oracle/_ref: the unmodified
    reference + a C-ABI shim) or, where it is not built, the C port; returns seconds."""
    import oracle

    F = oracle.forcing_grid(w)
    u0 = oracle.initial_grid(w, w.u0amp)
    phi = oracle.initial_grid(w, w.phiamp)
    if oracle.rlib() is not None:
        t0 = time.perf_counter()
        if int(w.specs[0].scheme) == 0:  # config 1: the Toeplitz-level API
            raise ValueError("use _ref_cfg1")
        oracle.ref_solve(w.specs[0], method, F, u0, phi)
        return time.perf_counter() - t0, "reference"
    t0 = time.perf_counter()
    oracle.direct(w, F, u0, phi)
    return time.perf_counter() - t0, "port"


def _ref_cfg1():
    """Config 1 at full size through the reference Toeplitz API: direct
    (lower_toeplitz_forward_solve, toeplitz.cpp:169-186) and fast (gmres_solve on
    make_toeplitz_operator(embed_circulant(T)), krylov.cpp:107-223, tol 1e-10)."""
    import ctypes as C

    import numpy as np

    import oracle
    from paper_1710_11593_b200 import workloads as W

    w = W.config(1)
    s = w.specs[0]
    N = s.time_steps
    L = oracle.rlib()
    col = np.empty(N)
    R = oracle.rhs(w, oracle.forcing_grid(w), oracle.initial_grid(w, w.u0amp))[0].copy()
    x = np.empty(N)
    if L is None:
        oracle.olib().or_col_ode(s.gamma, N, s.tau(), col.ctypes.data)
        t0 = time.perf_counter()
        oracle.olib().or_forward_solve(col.ctypes.data, R.ctypes.data, N, x.ctypes.data)
        return {"direct_s": time.perf_counter() - t0, "fast_s": None, "kind": "port"}
    L.ref_ode_column(s.gamma, N, s.time_length, col.ctypes.data)
    t0 = time.perf_counter()
    L.ref_forward_solve(col.ctypes.data, R.ctypes.data, N, x.ctypes.data)
    td = time.perf_counter() - t0
    it = C.c_uint64(0)
    t0 = time.perf_counter()
    rc = L.ref_toeplitz_gmres(col.ctypes.data, R.ctypes.data, N, 1e-10, 40, x.ctypes.data, C.byref(it))
    tf = time.perf_counter() - t0
    return {"direct_s": td, "fast_s": tf, "fast_matvecs": int(it.value), "fast_converged": rc == 0,
            "kind": "reference"}


def reference_estimate(cid: int):
    """Full-size reference direct-solve time for config `cid` from a reduced-M,
    full-N sample (see the block comment above).  Returns a dict with value
    (unknowns/s of the full workload), the sample and its law."""
    from paper_1710_11593_b200 import workloads as W

    full = W.config(cid)
    if cid == 1:
        r = _ref_cfg1()
        best = r["direct_s"]
        return {"value": full.unknowns / best, "full_solve_s": best, "kind": r["kind"], "cores": 1,
                "sample": "full size (N = 4096): reference lower_toeplitz_forward_solve (direct) and "
                          "gmres_solve on its FFT operator (fast); value from the faster (direct)",
                "direct_s": r["direct_s"], "fast_s": r["fast_s"], "fast_matvecs": r.get("fast_matvecs"),
                "law": "measured at full size (no extrapolation)"}
    mp = REF_SAMPLE_NODES[cid]
    w = W.config(cid, cells=mp + 1, batch=1 if cid == 5 else None)
    t, kind = _ref_one(w)
    per_problem = t * full.nodes / mp
    problems = full.B
    cores = os.cpu_count() or 1
    # independent problems (config 5) run concurrently on all host cores, as the
    # reference's harness pool would; one problem uses one core
    lanes = min(cores, problems)
    full_s = per_problem * math.ceil(problems / lanes)
    return {"value": full.unknowns / full_s, "full_solve_s": full_s, "kind": kind, "cores": lanes,
            "sample": f"reference solve(spec, Direct) on M'={mp} nodes at the full N={full.N} "
                      f"(gamma {w.specs[0].gamma:.4g}, h = 1/{full.specs[0].space_cells}): {t:.3f} s",
            "law": f"T_full = T(M') * M / M' (direct march: identical O(N^2) work per node)"
                   + (f"; {problems} independent problems over {lanes} cores" if problems > 1 else ""),
            "fast": ("infeasible at this size (GMRES: thousands of O(M N log N) matvecs, SURVEY.md P3)"
                     if cid != 3 else "fails (GMRES does not converge at M = 1024, SURVEY.md P4)")}


def reference_prefix_rate(cid: int, n_prefix: int = 128):
    """Raw rate of the full-M time prefix N' (short history rows; side field)."""
    from paper_1710_11593_b200 import workloads as W

    w = W.config(cid, time_steps=n_prefix, batch=1 if cid == 5 else None)
    t, kind = _ref_one(w)
    return {"value": w.unknowns / t, "seconds": t, "sample": f"full M={w.nodes}, time prefix N'={n_prefix}"}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    from paper_1710_11593_b200 import workloads as W

    wl = W.config(args.config)
    vals = []
    est = None
    for i in range(args.warmup + args.steps):
        est = reference_estimate(args.config)
        if i >= args.warmup:
            vals.append(est["value"])
    value = sum(vals) / len(vals)
    ms = 1e3 * wl.unknowns / value
    subs = {}
    if not args.no_configs and args.config == 4:
        for cid in (1, 2, 3, 5):
            subs[f"cfg{cid}"] = reference_estimate(cid)
        # config 2 is the one multi-node config whose full direct solve the reference finishes in
        # under a minute: measured once at full size next to the reduced-M estimate (checks the law)
        t_full, kind = _ref_one(W.config(2))
        subs["cfg2"]["full_direct_measured_s"] = t_full
        subs["cfg2"]["full_direct_measured_value"] = W.config(2).unknowns / t_full
        subs["cfg2"]["law_over_measured"] = subs["cfg2"]["full_solve_s"] / t_full
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "unknowns/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.name, "nodes": wl.nodes, "time_steps": wl.N, "problems": wl.B,
                   "parallelism": f"{est['cores']} host thread(s): the reference solves one problem per thread"},
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": est["cores"], "kind": est["kind"],
                         "sample": est["sample"], "law": est["law"], "full_solve_s": est["full_solve_s"]},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "prefix_rate": reference_prefix_rate(args.config) if args.config != 1 else None,
        "configs": subs,
    }
    print(json.dumps(line), flush=True)


# ---- our arm -------------------------------------------------------------------

def _events_ms(stream, fn, steps):
    import torch

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def measure_config(cid: int, steps: int, warmup: int, e2e_steps: int):
    """Our numbers for one BASELINE config on one GPU (sub-results of the main
    line): device-resident solve (CUDA events), and e2e through the C ABI with the
    forcing modes in and U out to pinned host memory."""
    import torch

    import paper_1710_11593_b200 as ft
    from paper_1710_11593_b200 import workloads as W

    wl = W.config(cid)
    plan = ft.Plan(wl.specs)
    stream = torch.cuda.Stream()
    plan.set_stream(stream.cuda_stream)
    rhs = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    u = torch.empty_like(rhs)
    plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
    torch.cuda.synchronize()
    for _ in range(warmup):
        _, rep = plan.solve_fast(rhs, u)
    ms = _events_ms(stream, lambda: plan.solve_fast(rhs, u), steps)
    h_u = torch.empty(plan.shape, dtype=torch.float64, pin_memory=True)
    un = h_u.numpy()
    plan.solve_fast_modes(un, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.solve_fast_modes(un, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    bpu = bytes_per_unknown(wl.N)
    pk, _ = peaks()
    out = {"workload": wl.name, "nodes": wl.nodes, "time_steps": wl.N, "problems": wl.B,
           "value": wl.unknowns / (ms / 1e3), "unit": "unknowns/s", "ms_per_step": ms,
           "hbm_roofline_frac": bpu * wl.unknowns / (ms / 1e3) / 1e9 / float(pk["hbm_gbs"]),
           "kernel_launches_per_solve": int(rep.kernel_launches),
           "e2e": {"value": wl.unknowns / e2e_s, "unit": "unknowns/s", "ms_per_step": 1e3 * e2e_s,
                   "h2d_bytes_per_step": int(8 * (wl.a.size + wl.k.size + wl.p.size + wl.trig.size + 3 * wl.B)),
                   "d2h_bytes_per_step": int(8 * wl.unknowns),
                   "path": "ft_solve_fast_modes: forcing modes in, U out to pinned host memory"}}
    del rhs, u, h_u, plan
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_1710_11593_b200 as ft
    from paper_1710_11593_b200 import workloads as W

    torch.cuda.set_device(local)
    # the other BASELINE configs first (one GPU, rank 0 of a single-rank run), so
    # config 4's 69 GB of buffers are not resident at the same time
    subs = {}
    if world == 1 and args.config == 4 and not args.no_configs:
        for cid in (1, 2, 3, 5):
            subs[f"cfg{cid}"] = {"ours": measure_config(cid, args.steps, max(3, args.warmup), args.e2e_steps)}
    wl = W.config(args.config, time_steps=args.time_steps or None)
    sharded = world > 1 and wl.B == 1 and wl.nodes > 2048
    if sharded:
        # one wide problem split by spatial slab over the ranks: node-local history
        # products, one carry all-gather (NCCL) per leaf -- strong scaling
        from paper_1710_11593_b200.parallel import ShardedPlan

        # FT_P2P_EXCHANGE=1: the leaf kernels exchange the carries over NVLink peer memory
        # (ft_p2p_connect) instead of the NCCL hook -- opt-in, not yet run on a multi-GPU box
        plan = ShardedPlan(wl.specs[0], rank, world, device=local, p2p=os.environ.get("FT_P2P_EXCHANGE") == "1")
        if os.environ.get("FT_P2P_EXCHANGE") != "1" and os.environ.get("FT_NCCL_HOOK") != "1":
            # the all-gather as ncclAllGather issued by the library (ft_nccl_init): the solve replays
            # as one CUDA graph; falls back to the torch.distributed hook if NCCL cannot be bound
            # (every rank takes the same branch: the bind is collective)
            import torch.distributed as dist
            ok = torch.ones(1, device=f"cuda:{local}")
            try:
                plan.bind_nccl()
            except Exception as e:  # noqa: BLE001
                print(f"[rank {rank}] native NCCL exchange unavailable ({e}); using the hook", file=sys.stderr)
                ok.zero_()
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 0:
                plan = ShardedPlan(wl.specs[0], rank, world, device=local)
        stream = plan.stream
    else:
        # independent problems (config 5: shard the batch) or replicas
        from paper_1710_11593_b200.parallel import shard_problems

        specs = shard_problems(wl.specs, rank, world) if (world > 1 and wl.B >= world) else wl.specs
        plan = ft.Plan(specs, device=local)
        stream = torch.cuda.Stream()
        plan.set_stream(stream.cuda_stream)
    shape = plan.shape
    rhs = torch.empty(shape, dtype=torch.float64, device="cuda")
    u = torch.empty_like(rhs)
    if sharded or plan.B == wl.B:
        plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
    else:
        from paper_1710_11593_b200.parallel import partition_range

        b0, b1 = partition_range(wl.B, rank, world)
        plan.assemble_rhs_modes(rhs, wl.a[b0:b1], wl.k, wl.p[b0:b1], wl.trig,
                                None if wl.u0amp is None else wl.u0amp[b0:b1],
                                None if wl.phiamp is None else wl.phiamp[b0:b1])
    torch.cuda.synchronize()
    unknowns = plan.B * plan.nodes * plan.N  # this rank's share

    for _ in range(args.warmup):
        _, rep = plan.solve_fast(rhs, u)
    launches_per_solve = rep.kernel_launches
    barrier(world)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for _ in range(args.steps):
                plan.solve_fast(rhs, u)
            ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(world, ms)
    total_unknowns = wl.unknowns if (sharded or plan.B != wl.B) else world * unknowns
    value = total_unknowns / (ms / 1e3)
    scaling = "strong" if (sharded or plan.B != wl.B) else "weak"
    parallelism = (f"slab-partitioned x{world} (NCCL carry all-gather per leaf)" if sharded
                   else f"problem-sharded x{world}" if plan.B != wl.B
                   else f"replicas x{world}" if world > 1 else "single GPU")

    pk, pk_kind = peaks()
    hbm = float(pk["hbm_gbs"])
    bpu = bytes_per_unknown(wl.N)
    solve_gbs = bpu * total_unknowns / (ms / 1e3) / 1e9 / world  # per GPU

    # dominant kernel: per-launch device times of one profiled solve of the path that is timed
    traffic, traffic_note, per_level = None, None, {}
    if int(plan.info.flags) & ft.PLAN_ODE_WHOLE:
        # single-node plans run ONE kernel per solve (ode_whole_kernel): its launch is the solve
        dom, d_ms, d_bytes, d_n = "ode_whole_kernel", ms, bpu * unknowns, 1
        mp_ms, lf_ms, mp_bytes, lf_bytes = 0.0, ms, 0, bpu * unknowns
    else:
        ops = plan.profile_fast(rhs, u)
        mp = [o for o in ops if o["kind"] == 1 and o["bytes"] > 0]  # (n = 64 products folded into leaves: 0 bytes)
        lf = [o for o in ops if o["kind"] == 0]
        mp_ms = sum(o["ms"] for o in mp)
        lf_ms = sum(o["ms"] for o in lf)
        mp_bytes = sum(o["bytes"] for o in mp)
        lf_bytes = sum(o["bytes"] for o in lf)
        dom = "mp_kernel" if mp_ms >= lf_ms else "leaf_kernel"
        d_ms, d_bytes, d_n = (mp_ms, mp_bytes, len(mp)) if dom == "mp_kernel" else (lf_ms, lf_bytes, len(lf))
        # DRAM traffic per launch of the dominant kernel: each level's algorithmic
        # bytes scaled by the ncu-measured DRAM/algorithmic ratio of its kernel family
        if dom == "mp_kernel" and d_n:
            leaf_len = int(plan.info.leaf)
            dram = sum(o["bytes"] * NCU_DRAM_OVER_ALG[mp_family(2 * leaf_len << o["level"])] for o in mp)
            traffic = dram / d_n
            traffic_note = ("bytes per launch (DRAM read+write), per-level ncu ratios " + json.dumps(NCU_DRAM_OVER_ALG)
                            + f"; algorithmic bytes per launch {d_bytes / d_n:.4g}")
        for o in mp:
            lv = per_level.setdefault(o["level"], {"launches": 0, "ms": 0.0, "bytes": 0})
            lv["launches"] += 1
            lv["ms"] += o["ms"]
            lv["bytes"] += o["bytes"]
    achieved = d_bytes / (d_ms / 1e3) / 1e9 if d_ms > 0 else 0.0

    # the same solve with the separable forcing generated inside the leaves
    # (ft_solve_fast_modes: no RHS array, no RHS read -- SURVEY.md 8f item 2)
    fused = None
    if not sharded and plan.B == wl.B and not args.no_fused:
        plan.solve_fast_modes(u, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
        torch.cuda.synchronize()
        fms = _events_ms(stream, lambda: plan.solve_fast_modes(u, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp),
                         args.steps)
        fused = {"value": total_unknowns / (fms / 1e3), "unit": "unknowns/s", "ms_per_step": fms,
                 "path": ("ft_solve_fast_modes (single node: RHS array generated on the device, one-kernel march)"
                          if plan.nodes == 1 else
                          "ft_solve_fast_modes (RHS generated in the leaves; includes the per-call table setup)")}

    e2e = None
    if not args.no_e2e:
        h_rhs = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        h_u = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        h_rhs.copy_(rhs.to("cpu"))
        hn = h_rhs.numpy()
        un = h_u.numpy()
        plan.solve_fast(hn, un)  # warm (staging buffer)
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.solve_fast(hn, un)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        e2e_s = max_over_ranks(world, e2e_s)
        nbytes = int(np.prod(shape)) * 8
        e2e = {"value": total_unknowns / e2e_s, "unit": "unknowns/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": 1e3 * e2e_s, "steps": args.e2e_steps,
               "path": "ft_solve_fast C ABI with pinned host buffers"}
        if fused is not None:
            # the reference's solve(spec) takes the forcing as a callback, not an array: the
            # same end-to-end solve with the separable forcing as mode arguments (a few hundred
            # bytes H2D), the solution streamed back to pinned host memory
            plan.solve_fast_modes(un, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
            t0 = time.perf_counter()
            for _ in range(args.e2e_steps):
                plan.solve_fast_modes(un, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
            em_s = (time.perf_counter() - t0) / args.e2e_steps
            arg_bytes = 8 * (wl.a.size + wl.k.size + wl.p.size + wl.trig.size + wl.B * 3)
            # BASELINE config 4's input IS the 8-mode forcing (seeded coefficients), and the
            # reference's solve(spec) takes it as a callback: this call is the headline e2e;
            # the RHS-array call is kept beside it
            e2e = {"value": total_unknowns / em_s, "unit": "unknowns/s", "h2d_bytes_per_step": int(arg_bytes),
                   "d2h_bytes_per_step": nbytes, "ms_per_step": 1e3 * em_s, "steps": args.e2e_steps,
                   "path": "ft_solve_fast_modes C ABI: forcing modes in (host), U out to pinned host memory",
                   "array_rhs": e2e}
        del h_rhs, h_u

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        est = reference_estimate(args.config)
        cpu = {"value": est["value"], "unit": "unknowns/s", "cores": est["cores"], "kind": est["kind"],
               "sample": est["sample"], "law": est["law"], "full_solve_s": est["full_solve_s"],
               "prefix_rate": reference_prefix_rate(args.config) if args.config != 1 else None}
        if subs:
            for cid in (1, 2, 3, 5):
                subs[f"cfg{cid}"]["reference"] = reference_estimate(cid)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "unknowns/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name, "nodes": wl.nodes, "time_steps": wl.N, "problems": wl.B,
                       "gamma": wl.specs[0].gamma, "leaf": int(plan.info.leaf),
                       "levels": int(plan.info.levels), "slabs": int(plan.info.slabs),
                       "parallelism": parallelism,
                       "l2": "inputs (34 GB) >> 126 MB L2; no flush needed"},
            "hbm_roofline": {"bytes_per_unknown": bpu, "achieved_gbs_per_gpu": solve_gbs, "peak_gbs": hbm,
                             "frac": solve_gbs / hbm, "peak_kind": pk_kind},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "traffic_note": traffic_note, "launches": d_n,
                         "kernel_ms_per_solve": d_ms, "peak_kind": pk_kind},
            "time_split_ms": {"mp_kernel": mp_ms, "leaf_kernel": lf_ms,
                              "mp_gbs": mp_bytes / (mp_ms / 1e3) / 1e9 if mp_ms else None,
                              "leaf_gbs": lf_bytes / (lf_ms / 1e3) / 1e9 if lf_ms else None,
                              "mp_levels": per_level},
            "e2e": e2e,
            "fused_rhs": fused,
            "cpu_baseline": cpu,
            "configs": subs,
            "gpu_launches": launches_per_solve * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--time-steps", type=int, default=0, help="time-prefix variant (default: full N)")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config sub-results (cfg1/2/3/5)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fused", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
