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
built from /root/reference by oracle/build_ref.sh) on a bounded sample of the
same workload using all host cores.
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


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


# DRAM bytes / algorithmic bytes of one history-product launch, measured with
# ncu --set full on B200 (profiles/ncu_r01/kernels.json): direct kernel
# (n <= 128: 0.67), group-private single-CTA FFT (256 <= n <= 4096: 0.81 at
# n = 256, 0.90 at n = 512), 2- and 4-CTA clusters (n = 8192, 16384: 1.00),
# split K-branch kernels + combine with the branch scratch round trip
# (n >= 32768: 2.15 at K = 8; the pre-folded K = 16 level is taken equal).
NCU_DRAM_OVER_ALG = {"direct": 0.67, "single": 0.86, "cluster": 1.00, "split": 2.15}


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

def reference_sample(cid: int, n_prefix: int, threads: int):
    """One bounded sample: `threads` concurrent runs of the unmodified reference
    direct solver (the only reference path that runs at this size; its GMRES fast
    path is infeasible) on the time prefix N' of the workload at
    full M (tau = 1/N bit-exactly).  Returns (unknowns/s, seconds, info)."""
    import numpy as np

    import oracle
    from paper_1710_11593_b200 import workloads as W

    L = oracle.rlib()
    kind = "reference"
    if L is None:
        kind = "port"
    w = W.config(cid, time_steps=n_prefix)
    F = oracle.forcing_grid(w)
    u0 = oracle.initial_grid(w, w.u0amp)
    s = w.specs[0]
    res = [None] * threads

    def run(i):
        t0 = time.perf_counter()
        if kind == "reference":
            oracle.ref_solve(s, "direct", F, u0)
        else:
            oracle.direct(w, F, u0)
        res[i] = time.perf_counter() - t0

    t0 = time.perf_counter()
    ths = [threading.Thread(target=run, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    unknowns = threads * w.nodes * n_prefix
    return unknowns / wall, wall, {"kind": kind, "nodes": w.nodes, "n_prefix": n_prefix}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    n_prefix = args.ref_prefix
    vals = []
    for i in range(args.warmup + args.steps):
        v, wall, info = reference_sample(args.config, n_prefix, cores)
        if i >= args.warmup:
            vals.append((v, wall))
    value = sum(v for v, _ in vals) / len(vals)
    ms = 1e3 * sum(w for _, w in vals) / len(vals)
    from paper_1710_11593_b200 import workloads as W

    wl = W.config(args.config)
    N = wl.N
    # O(M N^2) direct-march law from the sample to the full size (labelled extrapolation)
    full_s = (ms / 1e3) * (N / n_prefix) ** 2  # each core ran one whole sample solve
    line = {
        "impl": "reference",
        "metric": "space-time unknowns solved/sec (M*N/s, fp64)",
        "value": value, "unit": "unknowns/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl.name, "nodes": wl.nodes, "time_steps": N, "problems": wl.B,
                   "sample_time_steps": n_prefix, "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "unknowns/s", "cores": cores, "kind": info["kind"],
                         "sample": f"{cores} concurrent reference direct solves of the time prefix "
                                   f"N'={n_prefix} at full M={wl.nodes} (tau = 1/{N} exactly); "
                                   f"the reference fast path (GMRES) is infeasible at this size",
                         "extrapolated_full_solve_s_one_core": full_s},
        "e2e": {"value": value, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---- our arm -------------------------------------------------------------------

def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_1710_11593_b200 as ft
    from paper_1710_11593_b200 import workloads as W

    torch.cuda.set_device(local)
    wl = W.config(args.config, time_steps=args.time_steps or None)
    sharded = world > 1 and wl.B == 1 and wl.nodes > 2048
    if sharded:
        # one wide problem split by spatial slab over the ranks: node-local history
        # products, one carry all-gather (NCCL) per leaf -- strong scaling
        from paper_1710_11593_b200.parallel import ShardedPlan

        # FT_P2P_EXCHANGE=1: the leaf kernels exchange the carries over NVLink peer memory
        # (ft_p2p_connect) instead of the NCCL hook -- opt-in, not yet run on a multi-GPU box
        plan = ShardedPlan(wl.specs[0], rank, world, device=local, p2p=os.environ.get("FT_P2P_EXCHANGE") == "1")
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

    # dominant kernel: per-launch device times of one profiled solve
    ops = plan.profile_fast(rhs, u)
    mp = [o for o in ops if o["kind"] == 1 and o["bytes"] > 0]  # (n = 64 products folded into leaves: 0 bytes)
    lf = [o for o in ops if o["kind"] == 0]
    mp_ms = sum(o["ms"] for o in mp)
    lf_ms = sum(o["ms"] for o in lf)
    mp_bytes = sum(o["bytes"] for o in mp)
    lf_bytes = sum(o["bytes"] for o in lf)
    dom = "mp_kernel" if mp_ms >= lf_ms else "leaf_kernel"
    d_ms, d_bytes, d_n = (mp_ms, mp_bytes, len(mp)) if dom == "mp_kernel" else (lf_ms, lf_bytes, len(lf))
    achieved = d_bytes / (d_ms / 1e3) / 1e9 if d_ms > 0 else 0.0
    # DRAM traffic per launch of the dominant kernel: each level's algorithmic
    # bytes scaled by the ncu-measured DRAM/algorithmic ratio of its kernel family
    traffic, traffic_note = None, None
    if dom == "mp_kernel" and d_n:
        leaf_len = int(plan.info.leaf)
        dram = sum(o["bytes"] * NCU_DRAM_OVER_ALG[mp_family(2 * leaf_len << o["level"])] for o in mp)
        traffic = dram / d_n
        traffic_note = ("bytes per launch (DRAM read+write), per-level ncu ratios " + json.dumps(NCU_DRAM_OVER_ALG)
                        + f"; algorithmic bytes per launch {d_bytes / d_n:.4g}")
    per_level = {}
    for o in mp:
        lv = per_level.setdefault(o["level"], {"launches": 0, "ms": 0.0, "bytes": 0})
        lv["launches"] += 1
        lv["ms"] += o["ms"]
        lv["bytes"] += o["bytes"]

    # the same solve with the separable forcing generated inside the leaves
    # (ft_solve_fast_modes: no RHS array, no RHS read -- SURVEY.md 8f item 2)
    fused = None
    if not sharded and plan.B == wl.B and not args.no_fused:
        plan.solve_fast_modes(u, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            f0.record(stream)
            for _ in range(args.steps):
                plan.solve_fast_modes(u, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
            f1.record(stream)
        torch.cuda.synchronize()
        fms = f0.elapsed_time(f1) / args.steps
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
        cores = os.cpu_count() or 1
        v, wall, info = reference_sample(args.config, args.ref_prefix, cores)
        cpu = {"value": v, "unit": "unknowns/s", "cores": cores, "kind": info["kind"],
               "sample": f"{cores} concurrent reference direct solves (oracle/_ref) of the time prefix "
                         f"N'={args.ref_prefix} at full M={wl.nodes}; wall {wall:.2f} s",
               "extrapolated_full_solve_s_one_core": wall * (wl.N / args.ref_prefix) ** 2,
               "extrapolation": "O(M N^2) direct-march law from the N' sample (one solve per core)"}

    if rank == 0:
        line = {
            "metric": "space-time unknowns solved/sec (M*N/s, fp64) and % of HBM roofline",
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
    ap.add_argument("--ref-prefix", type=int, default=128)
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
