"""Experiment driver: a config-4-shaped fast solve (optional time prefix / reduced M),
median solve time over a few repeats, the per-level split from ft_profile_fast, the
CTA-0 clock stamps of the last slab leaf (FT_LEAF_DBG=4) and a parity check of the
fast path against the on-device reference-order march on a small prefix."""
import sys; sys.path.insert(0, '.')
import argparse, ctypes as C, collections, statistics, torch
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--time-steps", type=int, default=0)
ap.add_argument("--cells", type=int, default=0)
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--split", action="store_true")
ap.add_argument("--nccl", action="store_true", help="one-rank NCCL exchange (two-kernel leaf + ncclAllGather in the graph)")
ap.add_argument("--check", type=int, default=0, help="parity vs ft_solve_direct on this many steps (0: off)")
a = ap.parse_args()
wl = W.config(a.config, time_steps=a.time_steps or None, cells=a.cells or None)
plan = ft.Plan(wl.specs, device=0)
if a.nccl:
    plan.nccl_init(ft.nccl_unique_id(), 0, 1)
rhs = torch.empty(plan.shape, dtype=torch.float64, device="cuda"); u = torch.empty_like(rhs)
plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
ms = []
for _ in range(a.solves):
    _, rep = plan.solve_fast(rhs, u)
    ms.append(rep.device_ms)
print(f"solve ms median {statistics.median(ms):.3f} min {min(ms):.3f} (launches {rep.kernel_launches})")
clk = (C.c_longlong * 16)()
if ft.lib().ft_debug_leaf_clocks(plan._h, clk) == 0:
    c = list(clk)
    names = [(12, 8, "entry->pdl"), (8, 15, "stage R"), (15, 5, "stage U (fuse0)"), (5, 9, "fuse0 product"),
             (15, 9, "stage->steps (total)"), (9, 10, "step loop"), (10, 11, "publish"), (11, 14, "to barrier"),
             (14, 13, "grid barrier"), (13, 0, "to correct"), (0, 1, "load carries"), (1, 2, "phase 2"),
             (2, 3, "phase 3"), (3, 4, "store"), (12, 4, "TOTAL")]
    print("leaf stamps (cycles):", ", ".join(f"{n} {c[j] - c[i]}" for i, j, n in names if c[i] and c[j]))
if a.split:
    ops = plan.profile_fast(rhs, u)
    lv = collections.defaultdict(float); cnt = collections.Counter()
    for o in ops:
        key = "leaf" if o["kind"] == 0 else f"n={64 << o['level']}"
        lv[key] += o["ms"]; cnt[key] += 1
    print("split:", ", ".join(f"{k}: {v:.2f} ms/{cnt[k]}" for k, v in lv.items()), f"| sum {sum(lv.values()):.2f}")
if a.check:
    wc = W.config(a.config, time_steps=a.check, cells=a.cells or None)
    pc = ft.Plan(wc.specs, device=0)
    r = torch.empty(pc.shape, dtype=torch.float64, device="cuda")
    pc.assemble_rhs_modes(r, wc.a, wc.k, wc.p, wc.trig, wc.u0amp, wc.phiamp)
    uf, _ = pc.solve_fast(r); ud, _ = pc.solve_direct(r)
    err = ((uf - ud).abs().max() / ud.abs().max()).item()
    print(f"check N'={a.check}: fast vs direct march max rel {err:.3e}", "OK" if err <= 1e-10 else "FAIL")
