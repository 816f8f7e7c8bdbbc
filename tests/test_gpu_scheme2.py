"""Scheme 2 (hyperbolic transport, 0 < gamma < 1; reference schemes.cpp:149-266)
on the GPU through the C ABI, against the CPU oracle (bitwise equal to the
unmodified reference, test_oracle.py) and the reference's golden fixtures.

The D&C treats Scheme 2 as the upwind BLTT system  A~_0 U_i - B~_0 U_(i-1) = r
whose history (B~_j = -A~_j for j >= 1, schemes.cpp:162-165) acts on
U_i + U_(i-1): the leaf pushes the stencil sum, the history products read
V = U_i + U_(i-1).  Tolerance (north_star): <= 1e-10 max-normwise relative."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_1710_11593_b200 import workloads as W

pytestmark = pytest.mark.gpu
TOL = 1e-10
GOLD = Path(__file__).resolve().parent / "golden"


def _inputs(oracle, w):
    return oracle.forcing_grid(w), oracle.initial_grid(w, w.u0amp)


@pytest.mark.parametrize("gamma,steps,cells,u0amp", [
    (0.5, 16, 8, None),          # reference test_schemes.cpp:146-163 shape
    (0.1, 32, 16, None),         # test_schemes.cpp:137-143 gammas
    (0.9, 32, 16, None),
    (0.3, 1000, 33, 1.0),        # ragged leaf, u0 term
    (0.7, 4096, 257, -0.5),      # every FFT level up to n = 4096, 2 nodes per thread
    (0.2, 2048, 1025, 0.25),     # 4 nodes per thread, leaf 16
    (0.6, 1024, 2049, 1.0),      # widest single-slab problem (8 nodes per thread, leaf 8)
])
def test_fast_matches_oracle(ft, oracle_mod, gamma, steps, cells, u0amp):
    w = W.transport(gamma, steps, cells, u0amp)
    F, u0 = _inputs(oracle_mod, w)
    ref = oracle_mod.direct(w, F, u0)
    plan = ft.Plan(w.specs)
    R = plan.assemble_rhs_grid(F, u0)
    assert np.array_equal(R, oracle_mod.rhs(w, F, u0))  # Scheme2Rhs restated bitwise
    U, rep = plan.solve_fast(R)
    err = oracle_mod.relerr(U, ref)
    assert err <= TOL, f"rel err {err:.3e}"
    assert rep.kernel_launches > 0


def test_long_run_every_level(ft, oracle_mod):
    """N = 32768 on a few nodes: every D&C level including the cluster (n = 16384)
    and split K-branch (n = 32768) history products."""
    w = W.transport(0.4, 32768, 4, 1.0)
    F, u0 = _inputs(oracle_mod, w)
    plan = ft.Plan(w.specs)
    U, _ = plan.solve_fast(plan.assemble_rhs_grid(F, u0))
    assert oracle_mod.relerr(U, oracle_mod.direct(w, F, u0)) <= TOL


@pytest.mark.parametrize("gamma,steps,cells,u0amp", [(0.5, 16, 8, None), (0.3, 200, 33, 1.0),
                                                     (0.8, 128, 300, -1.0)])
def test_direct_gpu_is_reference_order(ft, oracle_mod, gamma, steps, cells, u0amp):
    """ft_solve_direct follows schemes.cpp:210-232 operation by operation
    (--fmad=false): bitwise equal to the reference."""
    w = W.transport(gamma, steps, cells, u0amp)
    F, u0 = _inputs(oracle_mod, w)
    plan = ft.Plan(w.specs)
    U, _ = plan.solve_direct(plan.assemble_rhs_grid(F, u0))
    assert np.array_equal(U, oracle_mod.direct(w, F, u0))


@pytest.mark.parametrize("name,kw", [("s2_g0.5_n16_m8", dict(gamma=0.5, time_steps=16, cells=8)),
                                     ("s2_g0.3_n64_m33_u0", dict(gamma=0.3, time_steps=64, cells=33, u0amp=1.0)),
                                     ("s2_g0.9_n100_m20_u0", dict(gamma=0.9, time_steps=100, cells=20, u0amp=-0.7))])
def test_fast_matches_reference_golden(ft, name, kw):
    g = np.load(GOLD / "golden.npz")
    w = W.transport(**kw)
    plan = ft.Plan(w.specs)
    u0 = g[f"{name}_u0"] if f"{name}_u0" in g else None
    U, _ = plan.solve_fast(plan.assemble_rhs_grid(g[f"{name}_F"], u0))
    ref = g[f"{name}_direct"]
    assert np.max(np.abs(U - ref)) / np.max(np.abs(ref)) <= TOL


def test_fast_reproduces_transport_table(ft, oracle_mod):
    """Reference acceptance criterion 5 (acceptance.cpp:241-250): Example 2 at
    tau = 2^-10, h = 2^-3..2^-8.  The frozen column carries the reference's
    documented x10 scale defect (proj/README.md:92-96): measured errors are one
    tenth of it (5%), rates within 0.05, fast == direct to 1e-10."""
    tables = json.loads((GOLD / "tables.json").read_text())
    for col in tables["kTransportReference"]:
        errs = []
        for e in range(3, 9):
            w = W.example(2, col["gamma"], e)
            w.specs[0].time_steps = 1 << 10
            F = oracle_mod.forcing_grid(w)
            plan = ft.Plan(w.specs)
            R = plan.assemble_rhs_grid(F)
            U, _ = plan.solve_fast(R)
            Ud, _ = plan.solve_direct(R)
            assert oracle_mod.relerr(U, Ud) <= TOL
            errs.append(W.l2_final(w, U))
        for i, err in enumerate(errs):
            assert abs(err - 0.1 * col["errors"][i]) <= 0.05 * 0.1 * col["errors"][i], (col["gamma"], i, err)
        for i in range(1, len(errs)):
            assert abs(math.log2(errs[i - 1] / errs[i]) - col["rates"][i - 1]) <= 0.05


def test_device_rhs_modes(ft, oracle_mod):
    """ft_assemble_rhs_modes for Scheme 2 (x = (i - 1/2) h, u0 at x_i and x_(i-1))
    against the host assembly from the oracle's glibc forcing grid (device libm:
    a few ulp)."""
    import torch

    w = W.transport(0.35, 300, 65, 0.8)
    F, u0 = _inputs(oracle_mod, w)
    plan = ft.Plan(w.specs)
    Rh = plan.assemble_rhs_grid(F, u0)
    Rd = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    plan.assemble_rhs_modes(Rd, w.a, w.k, w.p, w.trig, w.u0amp, None)
    assert oracle_mod.relerr(Rd.cpu().numpy(), Rh) <= 1e-14


@pytest.mark.parametrize("gamma,steps,cells,u0amp", [(0.5, 300, 1100, 1.0),   # 3 slabs, ragged last
                                                     (0.3, 96, 4097, -0.5),   # 8 slabs (cooperative leaf)
                                                     (0.8, 64, 2200, None)])
def test_wide_problems_slab_leaf(ft, oracle_mod, gamma, steps, cells, u0amp):
    """Problems wider than 512 nodes: the slab (SPIKE) leaf with the stencil-aware
    response tables (the injection is the left neighbour's boundary value, which also
    enters the first node's history) and V written from the corrected tile."""
    w = W.transport(gamma, steps, cells, u0amp)
    F, u0 = _inputs(oracle_mod, w)
    plan = ft.Plan(w.specs)
    assert plan.info.slabs > 1
    U, _ = plan.solve_fast(plan.assemble_rhs_grid(F, u0))
    assert oracle_mod.relerr(U, oracle_mod.direct(w, F, u0)) <= TOL
