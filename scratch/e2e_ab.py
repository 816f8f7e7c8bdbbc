"""e2e variants of ft_solve_fast_modes / ft_solve_fast with pinned host buffers (cfg4)."""
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
wl = W.config(4)
plan = ft.Plan(wl.specs, device=0)
hu = torch.empty(plan.shape, dtype=torch.float64, pin_memory=True).numpy()
plan.solve_fast_modes(hu, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
t0 = time.perf_counter()
for _ in range(3):
    plan.solve_fast_modes(hu, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
print("modes e2e ms", (time.perf_counter() - t0) / 3 * 1e3, flush=True)
