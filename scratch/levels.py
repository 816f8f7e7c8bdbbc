"""Per-level device times (ft_profile_fast) of one solve; prints one line per config/env."""
import sys, os; sys.path.insert(0, '.')
import argparse, collections, torch
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=4); ap.add_argument("--time-steps", type=int, default=0)
ap.add_argument("--tag", default=""); a = ap.parse_args()
wl = W.config(a.config, time_steps=a.time_steps or None)
plan = ft.Plan(wl.specs, device=0)
rhs = torch.empty(plan.shape, dtype=torch.float64, device="cuda"); u = torch.empty_like(rhs)
plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
plan.solve_fast(rhs, u)
ops = plan.profile_fast(rhs, u)
lv = collections.defaultdict(float); leaf = 0.0
for o in ops:
    if o["kind"] == 0: leaf += o["ms"]
    else: lv[o["level"]] += o["ms"]
_, rep = plan.solve_fast(rhs, u)
print(a.tag, "solve %.1f ms" % rep.device_ms, "leaf %.1f" % leaf, "mp %.1f" % sum(lv.values()),
      " ".join("%d:%.1f" % (k, v) for k, v in sorted(lv.items())), flush=True)
