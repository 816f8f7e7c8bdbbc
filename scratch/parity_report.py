"""Parity numbers for DESIGN.md / profiles: GPU fast path vs the oracle (reference-order fp64)
and vs the long-double march, on the BASELINE configs (full size or stated prefix)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, oracle
import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W
rows = []
def run(label, cid, kw, ld=False, rhs_mode=0):
    w = W.config(cid, **kw)
    F = oracle.forcing_grid(w); u0 = oracle.initial_grid(w, w.u0amp); phi = oracle.initial_grid(w, w.phiamp)
    t0 = time.perf_counter(); ref = oracle.direct(w, F, u0, phi, rhs_mode); tcpu = time.perf_counter() - t0
    plan = ft.Plan(w.specs, rhs_mode=rhs_mode)
    R = plan.assemble_rhs_grid(F, u0, phi)
    U, rep = plan.solve_fast(R)
    Ud, _ = plan.solve_direct(R) if w.nodes * w.N <= 2e7 and w.N <= 4096 else (None, None)
    r = dict(case=label, nodes=w.nodes, N=w.N, B=w.B, fast_vs_oracle=oracle.relerr(U, ref), cpu_oracle_s=tcpu)
    if Ud is not None: r["gpu_direct_vs_oracle"] = oracle.relerr(Ud, ref)
    if ld:
        Ul = np.vstack([oracle.march_ld(w.specs[b], R[b*w.nodes:(b+1)*w.nodes]) for b in range(w.B)])
        r["fast_vs_longdouble"] = oracle.relerr(U, Ul); r["oracle_vs_longdouble"] = oracle.relerr(ref, Ul)
    if w.exact and cid != 1: r["l2_error_vs_exact"] = W.l2_final(w, U)
    rows.append(r); print(json.dumps(r), flush=True)
run("cfg1 full (ODE, N=4096)", 1, {}, ld=True)
run("cfg2 full (M=256, N=16384)", 2, {})
run("cfg2 prefix N'=2048", 2, dict(time_steps=2048), ld=True)
run("cfg3 full M=1024, prefix N'=1024 (reference RHS)", 3, dict(time_steps=1024))
run("cfg3 node-prefix 16 nodes, full N=65536", 3, dict(cells=17))
run("cfg3 corrected-n1, 64 nodes, N'=512", 3, dict(time_steps=512, cells=65), ld=True, rhs_mode=1)
run("cfg4 full M=65536, prefix N'=128", 4, dict(time_steps=128), ld=True)
run("cfg4 full M=65536, prefix N'=512", 4, dict(time_steps=512))
run("cfg4 reduced M=64, full N=65536", 4, dict(cells=65))
run("cfg5 4 problems, prefix N'=4096", 5, dict(time_steps=4096, batch=4))
json.dump(rows, open('gpurun_out/parity_r01.json', 'w'), indent=1)
