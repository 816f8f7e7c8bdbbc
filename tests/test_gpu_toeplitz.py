"""GPU: the reference's structured-operator API (toeplitz.hpp) through the C ABI.

* ft_toeplitz_matvec / ft_block_matvec against the oracle's dense product (the
  reference's own oracle form, toeplitz.cpp:14-23) -- tight, the GPU sums
  directly -- and therefore within FFT rounding of the reference's
  toeplitz_matvec (pinned on CPU in test_oracle.py);
* ft_setup_toeplitz: the D&C (fast) and the reference's substitution order
  (direct, bitwise) for lower_toeplitz_forward_solve (toeplitz.cpp:169-186);
* the reference's error behaviour (zero diagonal, col0 != row0).
"""
import numpy as np
import pytest



def _dense_or(oracle_mod, col, row, x):
    y = np.empty_like(x)
    oracle_mod.olib().or_toeplitz_matvec(col.ctypes.data, row.ctypes.data, col.shape[0], x.ctypes.data, y.ctypes.data)
    return y


@pytest.mark.gpu
@pytest.mark.parametrize("n,count,lower", [(1, 1, False), (5, 3, False), (1000, 2, True), (4097, 1, False),
                                           (65536, 1, True)])
def test_toeplitz_matvec(ft, oracle_mod, n, count, lower):
    import torch

    col, row = oracle_mod.toeplitz_case(n, n, lower)
    X = np.random.default_rng(n).standard_normal((count, n))
    Y = ft.toeplitz_matvec(col, X, None if lower else row)
    ref = np.stack([_dense_or(oracle_mod, col, row, X[b]) for b in range(count)])
    scale = np.abs(col).sum() + np.abs(row).sum()
    assert np.max(np.abs(Y - ref)) <= 1e-14 * scale * np.max(np.abs(X))
    Xd = torch.from_numpy(X).cuda()
    Yd = ft.toeplitz_matvec(col, Xd, None if lower else row)  # device buffers
    assert np.array_equal(Yd.cpu().numpy(), Y)


@pytest.mark.gpu
def test_block_matvec(ft, oracle_mod):
    n, m, beta = 3000, 7, 0.41
    col, row = oracle_mod.toeplitz_case(n, 11)
    x = np.random.default_rng(4).standard_normal(n * m)
    y = ft.block_matvec(col, m, beta, x, row)
    ref = np.empty_like(x)
    oracle_mod.olib().or_block_matvec(col.ctypes.data, row.ctypes.data, n, m, beta, x.ctypes.data, ref.ctypes.data)
    scale = np.abs(col).sum() + np.abs(row).sum() + 2 * abs(beta)
    assert np.max(np.abs(y - ref)) <= 1e-14 * scale * np.max(np.abs(x))
    xi = x.copy()
    ft.lib().ft_block_matvec(col.ctypes.data, row.ctypes.data, n, m, beta, xi.ctypes.data, xi.ctypes.data)
    assert np.array_equal(xi, y)  # in place


@pytest.mark.gpu
@pytest.mark.parametrize("n,count", [(1, 1), (33, 2), (4096, 1), (20000, 3)])
def test_lower_toeplitz_solve(ft, oracle_mod, n, count):
    rng = np.random.default_rng(n)
    cols = np.stack([oracle_mod.toeplitz_case(n, n + b, True)[0] for b in range(count)])
    B = rng.standard_normal((count, n))
    plan = ft.Plan.toeplitz(cols)
    Xf, _ = plan.solve_fast(B)
    Xd, _ = plan.solve_direct(B)
    for b in range(count):
        xo = np.empty(n)
        assert oracle_mod.olib().or_forward_solve(cols[b].ctypes.data, B[b].ctypes.data, n, xo.ctypes.data) == 0
        assert np.array_equal(Xd[b], xo)  # reference summation order, bitwise
        assert oracle_mod.relerr(Xf[b], xo) <= 1e-10
    x1 = ft.lower_toeplitz_solve(cols[0], B[0])
    assert x1.shape == (n,) and np.array_equal(x1, Xf[0])


@pytest.mark.gpu
def test_toeplitz_errors(ft):
    with pytest.raises(ft.FractimeError, match="lower_toeplitz_forward_solve: zero diagonal"):
        ft.Plan.toeplitz(np.array([0.0, 1.0, 2.0]))
    with pytest.raises(ft.InvalidArgument, match="first_col\\[0\\] must equal first_row\\[0\\]"):
        ft.toeplitz_matvec(np.array([1.0, 2.0]), np.ones(2), np.array([3.0, 4.0]))
    plan = ft.Plan.toeplitz(np.array([2.0, 1.0]))
    with pytest.raises(ft.InvalidArgument, match="no scheme"):
        plan.assemble_rhs_grid(np.zeros((1, 2)))


@pytest.mark.gpu
@pytest.mark.parametrize("n,count", [(1000, 3), (65536, 2)])
def test_toeplitz_plan_apply_is_the_fft_matvec(ft, oracle_mod, n, count):
    """The O(n log n) route of toeplitz_matvec (embed_circulant + FFT, toeplitz.cpp:84-115) for
    lower-triangular operators applied many times: a Toeplitz plan (ft_setup_toeplitz) caches the
    level spectra and ft_apply runs the FFT history products.  Against the direct O(n^2) GPU
    product, which test_toeplitz_matvec pins to the oracle."""
    import torch

    cols = np.stack([oracle_mod.toeplitz_case(n, n + b, True)[0] for b in range(count)])
    X = np.random.default_rng(n).standard_normal((count, n))
    plan = ft.Plan.toeplitz(cols)
    Y = plan.apply(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = np.stack([ft.toeplitz_matvec(cols[b], X[b:b + 1])[0] for b in range(count)])
    scale = np.abs(cols).sum(axis=1).max() * np.abs(X).max()
    assert np.max(np.abs(Y - ref)) <= 1e-13 * scale


@pytest.mark.gpu
def test_random_toeplitz_operators_vs_dense(ft):
    """The reference's randomized operator checks (test_fft_toeplitz.cpp:76-103: 40 random
    Toeplitz matvecs, seed 42, 1e-13; acceptance criterion 2: 200 operators, seed 2024, 1e-12):
    200 random general Toeplitz operators of random size against the dense product."""
    rng = np.random.default_rng(2024)
    worst = 0.0
    for _ in range(200):
        n = int(rng.integers(1, 400))
        col = rng.standard_normal(n)
        row = rng.standard_normal(n)
        row[0] = col[0]
        x = rng.standard_normal((1, n))
        i, j = np.indices((n, n))
        T = np.where(i >= j, col[np.abs(i - j)], row[np.abs(i - j)])
        y = ft.toeplitz_matvec(col, x, row)[0]
        ref = T @ x[0]
        worst = max(worst, np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-300))
    assert worst <= 1e-12, worst


@pytest.mark.gpu
def test_plan_apply_scales_like_n_log_n(ft, oracle_mod):
    """The reference's complexity criterion for the FFT matvec (acceptance criterion 8: time
    ratio <= 2.6 per doubling of n, acceptance.cpp:293-348), on the plan route (ft_apply on a
    Toeplitz plan, 128 vectors at once), n = 16384 -> 32768 -> 65536."""
    import torch

    times = []
    for n in (16384, 32768, 65536):
        cols = np.tile(oracle_mod.toeplitz_case(n, 5, True)[0], (128, 1))
        plan = ft.Plan.toeplitz(cols)
        x = torch.randn(plan.shape, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        plan.apply(x, y)
        reps = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            plan.apply(x, y)
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        times.append(sorted(reps)[2])
        del plan, x, y
    print("ft_apply ms at n = 16384, 32768, 65536 (128 vectors):", times)
    assert times[1] / times[0] <= 2.6 and times[2] / times[1] <= 2.6, times
