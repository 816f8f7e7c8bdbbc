"""e2e timing of the streamed host path vs the serial path (config 4 or prefix)."""
import sys, os, time; sys.path.insert(0, '.')
import argparse, torch
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=4); ap.add_argument("--time-steps", type=int, default=0)
a = ap.parse_args()
wl = W.config(a.config, time_steps=a.time_steps or None)
plan = ft.Plan(wl.specs, device=0)
rhs = torch.empty(plan.shape, dtype=torch.float64, device="cuda"); u = torch.empty_like(rhs)
plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
_, rep = plan.solve_fast(rhs, u); print("device solve ms", rep.device_ms, flush=True)
hR = torch.empty(plan.shape, dtype=torch.float64, pin_memory=True); hR.copy_(rhs.cpu())
hU = torch.empty(plan.shape, dtype=torch.float64, pin_memory=True)
ref = u.cpu()
for tag, env in [("streamed", None), ("serial", "1")]:
    if env: os.environ["FT_NO_STREAM"] = env
    else: os.environ.pop("FT_NO_STREAM", None)
    plan.solve_fast(hR.numpy(), hU.numpy())
    t0 = time.perf_counter()
    for _ in range(2):
        _, rep = plan.solve_fast(hR.numpy(), hU.numpy())
    dt = (time.perf_counter() - t0) / 2
    err = (hU - ref).abs().max().item() / ref.abs().max().item()
    print(f"{tag}: e2e {dt*1e3:.1f} ms  ({wl.unknowns/dt:.3e} unknowns/s)  device_ms {rep.device_ms:.1f}  relerr vs device {err:.2e}", flush=True)
