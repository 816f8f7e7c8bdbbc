"""GPU parity: the CUDA fast / direct paths (through the C ABI) against the CPU
oracle (reference-order fp64 restatement, bitwise equal to the unmodified
reference -- see test_oracle.py) on identical seeded inputs.

Tolerance (north_star): max|U_gpu - U_ref| / max|U_ref| <= 1e-10 (fp64)."""
import numpy as np
import pytest

from paper_1710_11593_b200 import workloads as W

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _inputs(oracle, w, rhs_mode=0):
    F = oracle.forcing_grid(w)
    u0 = oracle.initial_grid(w, w.u0amp)
    phi = oracle.initial_grid(w, w.phiamp)
    return F, u0, phi


def _fast(ft, w, F, u0, phi, rhs_mode=0, **kw):
    plan = ft.Plan(w.specs, rhs_mode=rhs_mode, **kw)
    R = plan.assemble_rhs_grid(F, u0, phi)
    U, rep = plan.solve_fast(R)
    return plan, R, U, rep


CASES = [
    ("cfg1-full", 1, dict()),
    ("cfg1-odd", 1, dict(time_steps=1000)),
    ("cfg2-small", 2, dict(time_steps=512, cells=17)),
    ("cfg2-odd-nodes", 2, dict(time_steps=700, cells=32)),
    ("cfg2-prefix", 2, dict(time_steps=2048)),
    ("cfg3-small", 3, dict(time_steps=512, cells=17)),
    ("cfg3-prefix", 3, dict(time_steps=1024, cells=1025)),
    ("cfg4-reduced-M", 4, dict(time_steps=4096, cells=65)),
    ("cfg5-subset", 5, dict(time_steps=1024, batch=4)),
]


@pytest.mark.parametrize("name,cid,kw", CASES, ids=[c[0] for c in CASES])
def test_fast_matches_oracle(ft, oracle_mod, name, cid, kw):
    w = W.config(cid, **kw)
    F, u0, phi = _inputs(oracle_mod, w)
    ref = oracle_mod.direct(w, F, u0, phi)
    _, _, U, rep = _fast(ft, w, F, u0, phi)
    err = oracle_mod.relerr(U, ref)
    assert err <= TOL, f"{name}: rel err {err:.3e}"
    assert rep.kernel_launches > 0


@pytest.mark.parametrize("cid,kw", [(1, dict(time_steps=512)), (2, dict(time_steps=256, cells=33)),
                                    (3, dict(time_steps=256, cells=33)), (4, dict(time_steps=128, cells=65))])
def test_direct_gpu_is_reference_order(ft, oracle_mod, cid, kw):
    """ft_solve_direct marches in the reference's summation order with no FMA
    contraction: bitwise equal to the reference whenever u0 = 0 (the RHS is
    then formed identically), and within 1e-14 otherwise."""
    w = W.config(cid, **kw)
    F, u0, phi = _inputs(oracle_mod, w)
    ref = oracle_mod.direct(w, F, u0, phi)
    plan = ft.Plan(w.specs)
    R = plan.assemble_rhs_grid(F, u0, phi)
    U, rep = plan.solve_direct(R)
    if u0 is None:
        assert np.array_equal(U, ref)
    else:
        assert oracle_mod.relerr(U, ref) <= 1e-13


@pytest.mark.parametrize("cells,steps,slabs", [(4097, 96, 8), (3001, 100, 6), (2100, 64, 5)])
def test_multislab_leaf(ft, oracle_mod, cells, steps, slabs):
    """Problems wider than one CTA: slabs of 512 nodes, one carry exchange per
    leaf (phase 1 / reduced recursion / response-table correction), including
    an uneven last slab."""
    w = W.config(4, time_steps=steps, cells=cells)
    F, u0, phi = _inputs(oracle_mod, w)
    ref = oracle_mod.direct(w, F, u0, phi)
    plan, _, U, _ = _fast(ft, w, F, u0, phi)
    assert plan.info.slabs == slabs
    assert oracle_mod.relerr(U, ref) <= TOL
