"""One cfg4-shaped fast solve (optionally time-prefix) for ncu captures."""
import sys; sys.path.insert(0, '.')
import argparse, torch
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=4); ap.add_argument("--time-steps", type=int, default=0)
ap.add_argument("--solves", type=int, default=1); a = ap.parse_args()
wl = W.config(a.config, time_steps=a.time_steps or None)
plan = ft.Plan(wl.specs, device=0)
rhs = torch.empty(plan.shape, dtype=torch.float64, device="cuda"); u = torch.empty_like(rhs)
plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
for _ in range(a.solves):
    _, rep = plan.solve_fast(rhs, u)
print("solve ms", rep.device_ms, "launches", rep.kernel_launches)
