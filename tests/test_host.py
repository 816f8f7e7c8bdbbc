"""CPU: the C ABI library and host logic (no GPU compute).

* libfractime_b200.so loads and exports every entry point include/fractime_b200.h declares;
* without a CUDA device, setup fails loudly (FT_ECUDA) -- there is no CPU path;
* the divide-and-conquer schedule covers every (source, target) pair of the
  lower-triangular Toeplitz history exactly once (leaf: in-leaf lags; one
  history product per cross-leaf pair);
* the seeded workload generator agrees with the oracle's C implementation.
"""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1710_11593_b200 as ft
from paper_1710_11593_b200 import workloads as W

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    hdr = (ROOT / "include" / "fractime_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(ft_\w+)\s*\(", hdr, re.M)))


def test_abi_exports_every_declared_symbol():
    lib = ft.lib()
    syms = declared_symbols()
    assert len(syms) >= 14
    for name in syms:
        assert hasattr(lib, name), name
    assert set(ft.ABI_SYMBOLS) <= set(syms)


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ft.FractimeError) as e:
        ft.Plan(ft.ProblemSpec(ft.SchemeId.Diffusion, 0.5, 8, 4))
    assert e.value.code == -5 and "CUDA" in str(e.value)


def test_validation_messages():
    """Reference validate() wording (schemes.cpp:58-78) is raised before any device use."""
    with pytest.raises(ft.InvalidArgument, match="wave scheme needs gamma in \\(1, 2\\)"):
        ft.Plan(ft.ProblemSpec(ft.SchemeId.DiffusionWave, 0.5, 8, 4))
    with pytest.raises(ft.InvalidArgument, match="scheme needs gamma in \\(0, 1\\)"):
        ft.Plan(ft.ProblemSpec(ft.SchemeId.Diffusion, 1.5, 8, 4))
    with pytest.raises(ft.InvalidArgument, match="at least 2 space cells"):
        ft.Plan(ft.ProblemSpec(ft.SchemeId.Diffusion, 0.5, 8, 1))


def test_length_limit():
    """N beyond the history-product kernels fails at setup with FT_ELENGTH (the
    reference's std::length_error class), before any device use."""
    with pytest.raises(ft.FractimeError, match="at most 65536 time steps") as e:
        ft.Plan(ft.ProblemSpec(ft.SchemeId.Diffusion, 0.5, 65537, 4))
    assert e.value.code == -3


def test_buffer_checks_without_device():
    """The Python binding rejects wrong host buffers before the C ABI sees them."""
    from paper_1710_11593_b200 import _ptr

    with pytest.raises(ft.InvalidArgument, match="float64"):
        _ptr(np.zeros(4, dtype=np.float32))
    with pytest.raises(ft.InvalidArgument, match="contiguous"):
        _ptr(np.zeros((4, 4))[:, ::2])
    with pytest.raises(ft.InvalidArgument, match="elements"):
        _ptr(np.zeros(5), 4)
    assert _ptr(np.zeros(4), 4) != 0


@pytest.mark.parametrize("N,L", [(1, 32), (31, 32), (32, 32), (33, 32), (200, 32), (1000, 16), (4096, 32),
                                 (65536, 32), (777, 8)])
def test_schedule_covers_history_exactly_once(N, L):
    """Per target step t, the source intervals of the leaf (in-leaf lags) and of
    every history product targeting t are disjoint and tile [0, t) exactly; leaves
    run in time order and products only read solved steps."""
    ops = ft.schedule(N, L)
    intervals = [[] for _ in range(N)]
    solved = 0
    for op in ops:
        t0, ln = op["t0"], op["len"]
        if op["kind"] == 0:
            assert t0 == solved
            for t in range(t0, t0 + ln):
                intervals[t].append((t0, t))
            solved = t0 + ln
        else:
            h = L << op["level"]
            assert t0 == solved and t0 - h >= 0 and ln >= 1
            for t in range(t0, t0 + ln):
                intervals[t].append((t0 - h, t0))
    assert solved == N
    for t in range(N):
        iv = sorted(i for i in intervals[t] if i[1] > i[0])
        pos = 0
        for a, b in iv:
            assert a == pos, (t, iv)
            pos = b
        assert pos == t, (t, iv)


def test_splitmix_matches_oracle(oracle_mod):
    o = oracle_mod.olib()
    st = C.c_uint64(W.MASTER_SEED ^ 4)
    rng = W.SplitMix64(W.MASTER_SEED ^ 4)
    for _ in range(50):
        assert o.or_splitmix64(C.byref(st)) == rng.next()
    st = C.c_uint64(7)
    rng = W.SplitMix64(7)
    for _ in range(20):
        assert o.or_normal(C.byref(st)) == rng.normal()


def test_workload_shapes():
    w4 = W.config(4)
    assert (w4.B, w4.nodes, w4.N) == (1, 65536, 65536)
    assert w4.a.shape == (1, 8) and (1.0 <= w4.p).all() and (w4.p <= 3.0).all()
    w5 = W.config(5)
    assert (w5.B, w5.nodes, w5.N) == (64, 512, 32768)
    g = [s.gamma for s in w5.specs]
    assert min(g) > 0.1 and max(g) < 0.9
    w3 = W.config(3, time_steps=2048)
    assert w3.specs[0].tau() == 1.0 / 65536  # time-prefix keeps tau exact
    w3n = W.config(3, cells=17)
    assert w3n.specs[0].h() == 1.0 / 1025  # node-prefix keeps h exact


def test_harness_csv_format():
    """emit_csv restates the reference harness's CSV (harness.cpp:296-304)."""
    from paper_1710_11593_b200 import harness as H

    rows = [H.ConvergenceRow(3, 0.125, 0.125, 0.0084669, None, 0, 0.25, "fast", 0.1, "diffusion"),
            H.ConvergenceRow(4, 0.0625, 0.0625, 0.0021203, 1.9975, 0, 0.5, "fast", 0.1, "diffusion")]
    lines = H.emit_csv(rows).splitlines()
    assert lines[0] == "mesh_exp,h,tau,l2_error,rate,iterations,wall_seconds,method,gamma,scheme"
    assert lines[1] == "3,0.125,0.125,%.17g,,0,0.25,fast,0.10000000000000001,diffusion" % 0.0084669
    assert lines[2].split(",")[4] == "%.17g" % 1.9975
    assert H.exponent_ladder(3, 5) == [(3, 8, 8), (4, 16, 16), (5, 32, 32)]
    assert H.exponent_ladder(2, 3, 10) == [(2, 1024, 4), (3, 1024, 8)]
