"""CPU: pin the oracle (oracle/oracle.c) to the reference.

* bitwise against golden outputs the unmodified reference produced
  (tests/golden/make_golden.py, reference solve()/lower_toeplitz_forward_solve);
* against the reference's own known-answer tests (test_weights.cpp:10-59,
  acceptance.cpp criterion 1 and the frozen paper tables :72-90);
* bitwise against the live reference library when oracle/_ref is built.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_1710_11593_b200 import workloads as W

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD / "golden.npz")


def test_weight_kats(oracle_mod, gold):
    o = oracle_mod.olib()
    w = np.empty(4)
    o.or_weights(0.5, 4, w.ctypes.data)  # G(0.5): test_weights.cpp:10-18
    exp = [1.0, math.sqrt(2) - 1, math.sqrt(3) - math.sqrt(2), 2 - math.sqrt(3)]
    assert np.allclose(w, exp, rtol=1e-15, atol=0)
    assert np.array_equal(w, gold["weights_0_0.5_4"])
    m = np.empty(3)
    o.or_weights(0.5, 3, m.ctypes.data)  # M(1.5) uses p = 2 - 1.5: test_weights.cpp:20-26
    assert np.array_equal(m, gold["weights_1_1.5_3"])
    # tail form vs series (test_weights.cpp:50-59)
    p, k = 0.5, 1_000_000_000
    ref = p * k ** (p - 1) * (1 + (p - 1) / (2 * k) + (p - 1) * (p - 2) / (6 * k * k))
    assert abs(o.or_power_step(k, p) - ref) <= 1e-14 * ref
    assert o.or_power_step(k, p) == gold["power_step_1e9_0.5"][0]


@pytest.mark.parametrize("kind,gamma", [(0, 0.3), (1, 1.7)])
def test_weights_telescope(oracle_mod, gold, kind, gamma):
    """acceptance.cpp criterion 1: positive, decreasing, sum_{k<K} w_k = K^p."""
    o = oracle_mod.olib()
    p = (1.0 - gamma) if kind == 0 else (2.0 - gamma)  # as g_weights / m_weights form it
    w = np.empty(2000)
    o.or_weights(p, 2000, w.ctypes.data)
    assert (w > 0).all() and (np.diff(w) < 0).all()
    assert abs(w.sum() - 2000 ** p) <= 1e-12 * 2000 ** p
    key = f"weights_{kind}_{gamma}_2000"
    assert np.array_equal(w, gold[key])


CASES = ["cfg1_n256", "cfg2_m16_n128", "cfg2_m31_n100", "cfg3_m16_n128", "cfg4_m32_n64", "cfg4_m4096_n16",
         "s2_g0.5_n16_m8", "s2_g0.3_n64_m33_u0", "s2_g0.9_n100_m20_u0"]
CFG = {"cfg1_n256": (1, dict(time_steps=256)), "cfg2_m16_n128": (2, dict(time_steps=128, cells=17)),
       "cfg2_m31_n100": (2, dict(time_steps=100, cells=32)), "cfg3_m16_n128": (3, dict(time_steps=128, cells=17)),
       "cfg4_m32_n64": (4, dict(time_steps=64, cells=33)), "cfg4_m4096_n16": (4, dict(time_steps=16, cells=4097)),
       "s2_g0.5_n16_m8": ("transport", dict(gamma=0.5, time_steps=16, cells=8)),
       "s2_g0.3_n64_m33_u0": ("transport", dict(gamma=0.3, time_steps=64, cells=33, u0amp=1.0)),
       "s2_g0.9_n100_m20_u0": ("transport", dict(gamma=0.9, time_steps=100, cells=20, u0amp=-0.7))}


def case_workload(cid, kw):
    return W.transport(**kw) if cid == "transport" else W.config(cid, **kw)


@pytest.mark.parametrize("name", CASES)
def test_oracle_bitwise_vs_reference_golden(oracle_mod, gold, name):
    """The restated direct march is bit-identical to the reference's solve(Direct)."""
    cid, kw = CFG[name]
    w = case_workload(cid, kw)
    F = oracle_mod.forcing_grid(w)
    assert np.array_equal(F, gold[f"{name}_F"]), "forcing generator drifted"
    u0 = gold[f"{name}_u0"] if f"{name}_u0" in gold else None
    phi = gold[f"{name}_phi"] if f"{name}_phi" in gold else None
    U = oracle_mod.direct(w, F, u0, phi)
    assert np.array_equal(U, gold[f"{name}_direct"])


def test_oracle_vs_live_reference(oracle_mod):
    L = oracle_mod.rlib()
    if L is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for cid, kw in [(2, dict(time_steps=40, cells=9)), (3, dict(time_steps=33, cells=12)),
                    (4, dict(time_steps=17, cells=65)), ("transport", dict(gamma=0.4, time_steps=29, cells=13))]:
        w = case_workload(cid, kw)
        F = rng.standard_normal((w.nodes, w.N))
        u0 = rng.standard_normal(w.nodes + (1 if cid == "transport" else 0))
        phi = rng.standard_normal(w.nodes) if cid == 3 else None
        U = oracle_mod.direct(w, F, u0, phi)
        Ur, _, _ = oracle_mod.ref_solve(w.specs[0], "direct", F, u0, phi)
        assert np.array_equal(U, Ur)


@pytest.mark.parametrize("eid,key", [(4, "kDiffusionReference"), (3, "kWaveReference"),
                                     (2, "kTransportReference")])
def test_oracle_reproduces_paper_tables(oracle_mod, eid, key):
    """The reference's frozen Example 2/3/4 L2 errors (acceptance.cpp:62-90) at
    h = 2^-3..2^-6 (tau = h; Example 2: tau = 2^-10 fixed, acceptance.cpp:242),
    5% tolerance and rates within 0.05 as the reference checks.  The transport
    column carries the reference's documented x10 scale defect (proj/README.md:92-96):
    the measured errors equal one tenth of the frozen values."""
    tables = json.loads((GOLD / "tables.json").read_text())
    scale = 0.1 if eid == 2 else 1.0
    for col in tables[key]:
        errs = []
        for e in range(3, 7):
            w = W.example(eid, col["gamma"], e)
            if eid == 2:
                w.specs[0].time_steps = 1 << 10
            U = oracle_mod.direct(w, oracle_mod.forcing_grid(w))
            errs.append(W.l2_final(w, U))
        for i, err in enumerate(errs):
            assert abs(err - scale * col["errors"][i]) <= 0.05 * scale * col["errors"][i]
        for i in range(1, len(errs)):
            assert abs(math.log2(errs[i - 1] / errs[i]) - col["rates"][i - 1]) <= 0.05


def test_long_double_march_agrees(oracle_mod):
    """The long-double restatement (used for corrected-mode wave parity) agrees
    with the fp64 reference-order march to rounding on a benign case."""
    w = W.config(2, time_steps=64, cells=17)
    F = oracle_mod.forcing_grid(w)
    u0 = oracle_mod.initial_grid(w, w.u0amp)
    U = oracle_mod.direct(w, F, u0)
    R = oracle_mod.rhs(w, F, u0)
    Uld = oracle_mod.march_ld(w.specs[0], R)
    assert oracle_mod.relerr(U, Uld) < 1e-13


def test_scheme3_rhs_modes(oracle_mod):
    """Corrected mode differs from the reference only in the n = 1 row, by c*M0*u0."""
    w = W.config(3, time_steps=16, cells=9)
    F = oracle_mod.forcing_grid(w)
    u0 = oracle_mod.initial_grid(w, w.u0amp)
    phi = oracle_mod.initial_grid(w, w.phiamp)
    R0 = oracle_mod.rhs(w, F, u0, phi, 0)
    R1 = oracle_mod.rhs(w, F, u0, phi, 1)
    assert np.array_equal(R0[:, 1:], R1[:, 1:])
    mu = np.zeros(1)
    c = np.zeros(1)
    oracle_mod.olib().or_constants.argtypes = [__import__("ctypes").c_int, __import__("ctypes").c_double,
                                               __import__("ctypes").c_double, __import__("ctypes").c_void_p,
                                               __import__("ctypes").c_void_p]
    s = w.specs[0]
    oracle_mod.olib().or_constants(2, s.gamma, s.tau(), mu.ctypes.data, c.ctypes.data)
    assert np.allclose(R1[:, 0] - R0[:, 0], c[0] * u0, rtol=1e-12)


@pytest.mark.parametrize("n,lower", [(1, False), (7, False), (64, True), (300, False), (1025, True)])
def test_toeplitz_matvec_oracle_vs_reference(oracle_mod, n, lower):
    """or_toeplitz_matvec (dense, the reference's own oracle form) against the
    reference's FFT path (embed_circulant + toeplitz_matvec, toeplitz.cpp:84-115)."""
    r = oracle_mod.rlib()
    if r is None:
        pytest.skip("oracle/_ref not built")
    col, row = oracle_mod.toeplitz_case(n, n, lower)
    x = np.random.default_rng(1).standard_normal(n)
    y_or, y_ref = np.empty(n), np.empty(n)
    oracle_mod.olib().or_toeplitz_matvec(col.ctypes.data, row.ctypes.data, n, x.ctypes.data, y_or.ctypes.data)
    assert r.ref_toeplitz_matvec(col.ctypes.data, row.ctypes.data, n, x.ctypes.data, y_ref.ctypes.data) == 0
    dense = np.array([[row[j - i] if j >= i else col[i - j] for j in range(n)] for i in range(n)])
    assert np.allclose(y_or, dense @ x, rtol=0, atol=1e-13 * np.abs(dense).sum(1).max() * np.abs(x).max())
    assert np.max(np.abs(y_or - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))


def test_block_matvec_oracle_vs_reference(oracle_mod):
    r = oracle_mod.rlib()
    if r is None:
        pytest.skip("oracle/_ref not built")
    n, m, beta = 200, 5, -0.37
    col, row = oracle_mod.toeplitz_case(n, 3)
    x = np.random.default_rng(2).standard_normal(n * m)
    y_or, y_ref = np.empty(n * m), np.empty(n * m)
    oracle_mod.olib().or_block_matvec(col.ctypes.data, row.ctypes.data, n, m, beta, x.ctypes.data, y_or.ctypes.data)
    assert r.ref_block_matvec(col.ctypes.data, row.ctypes.data, n, m, beta, x.ctypes.data, y_ref.ctypes.data) == 0
    assert np.max(np.abs(y_or - y_ref)) <= 1e-12 * np.max(np.abs(y_ref))
