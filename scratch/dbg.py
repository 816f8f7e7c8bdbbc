import sys; sys.path.insert(0, '.')
import numpy as np, oracle
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
for cid, kw in [(2, dict(time_steps=1, cells=17)), (2, dict(time_steps=2, cells=17)), (2, dict(time_steps=32, cells=17)),
                (2, dict(time_steps=32, cells=33)), (2, dict(time_steps=64, cells=33)), (3, dict(time_steps=32, cells=17)),
                (3, dict(time_steps=64, cells=33))]:
    w = W.config(cid, **kw)
    F = oracle.forcing_grid(w); u0 = oracle.initial_grid(w, w.u0amp); phi = oracle.initial_grid(w, w.phiamp)
    ref = oracle.direct(w, F, u0, phi)
    plan = ft.Plan(w.specs)
    R = plan.assemble_rhs_grid(F, u0, phi)
    U, rep = plan.solve_fast(R)
    e = np.abs(U - ref)
    print(cid, kw, "err", oracle.relerr(U, ref), "first bad step", np.argmax(e.max(0) > 1e-10 * np.abs(ref).max()), "worst node", np.argmax(e.max(1)))
    if kw['time_steps'] <= 2:
        print(" U", U[:, 0][:6]); print(" ref", ref[:, 0][:6])
