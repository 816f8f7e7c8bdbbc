python scratch/levels.py --tag graph 2>&1 | tail -1
FT_NO_GRAPH=1 python scratch/levels.py --tag nograph 2>&1 | tail -1
python - <<'PY'
import sys, os, time; sys.path.insert(0, '.')
import torch, paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
for cid, ts in [(4, 0), (2, 0), (5, 0), (3, 0)]:
    wl = W.config(cid, time_steps=ts or None)
    plan = ft.Plan(wl.specs, device=0)
    rhs = torch.empty(plan.shape, dtype=torch.float64, device="cuda"); u = torch.empty_like(rhs)
    plan.assemble_rhs_modes(rhs, wl.a, wl.k, wl.p, wl.trig, wl.u0amp, wl.phiamp)
    res = {}
    for tag, env in [("graph", None), ("stream", "1")]:
        if env: os.environ["FT_NO_GRAPH"] = env
        else: os.environ.pop("FT_NO_GRAPH", None)
        plan.solve_fast(rhs, u)
        ts_ = []
        for _ in range(3):
            _, rep = plan.solve_fast(rhs, u); ts_.append(rep.device_ms)
        res[tag] = min(ts_)
        if tag == "graph": ug = u.clone()
    same = torch.equal(ug, u)
    print(f"cfg{cid}: graph {res['graph']:.2f} ms  stream {res['stream']:.2f} ms  bitwise-equal {same}", flush=True)
    del rhs, u, plan
PY
