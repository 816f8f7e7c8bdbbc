"""The plan's block system matrix on the GPU (ft_apply / ft_residual): the operator the
reference's fast path hands to GMRES (make_block_operator, src/toeplitz.cpp:194-201; applied
by block_matvec :150-167), here applied through the plan's own FFT history products.

* small shapes: against a dense numpy restatement of the same matrix (per node a lower
  triangular Toeplitz block in time from the plan's column, plus the spatial stencil);
* any size: the round trips  solve_fast(A x) = x  (forward error <= 1e-10) and
  A . solve_fast(R) = R  (backward error) -- size-independent properties, run at BASELINE
  config 4's full 65536 x 65536 (the solve and the operator share only the product kernels;
  the leaves, the slab coupling and the in-leaf windows are checked by them)."""
import numpy as np
import pytest

from paper_1710_11593_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _dense_apply(plan, w, x):
    """numpy: y[b, i, t] = sum_{j <= t} col_b[t - j] x[b, i, j] + stencil (reference block_matvec order)."""
    B = len(w.specs)
    nodes = plan.shape[0] // B
    N = plan.shape[1]
    y = np.zeros_like(x)
    for b, s in enumerate(w.specs):
        col = plan.column(b)
        T = np.zeros((N, N))
        for d in range(N):
            T += np.diag(np.full(N - d, col[d]), -d)
        xb = x[b * nodes:(b + 1) * nodes]
        yb = xb @ T.T
        h = s.h()
        if int(s.scheme) == 3:      # Scheme 4, tridiagonal: -(1/h^2) (x_(i-1) + x_(i+1)), Dirichlet
            off = 1.0 / (h * h)
            yb[1:] -= off * xb[:-1]
            yb[:-1] -= off * xb[1:]
        elif int(s.scheme) == 2:    # Scheme 3, upwind: -(1/h) x_(i-1)
            yb[1:] -= (1.0 / h) * xb[:-1]
        y[b * nodes:(b + 1) * nodes] = yb
    return y


@pytest.mark.parametrize("cid,kw", [
    (1, dict(time_steps=700)),
    (2, dict(time_steps=520, cells=33)),
    (3, dict(time_steps=300, cells=41)),            # wave scheme: exact near field (J = 64) inside the products
    (4, dict(time_steps=256, cells=1101)),          # 3 slabs
    (5, dict(time_steps=512, cells=65, batch=3)),
], ids=["ode", "diffusion", "wave", "diffusion-wide", "batch"])
def test_apply_matches_dense_operator(ft, cid, kw):
    import torch

    w = W.config(cid, **kw)
    plan = ft.Plan(w.specs)
    rng = np.random.default_rng(7 + cid)
    x = rng.standard_normal(plan.shape)
    y = plan.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = _dense_apply(plan, w, x)
    err = np.abs(y - ref).max() / np.abs(ref).max()
    assert err <= 1e-12, f"rel err {err:.3e}"
    assert np.array_equal(plan.apply(x), y)      # host arrays in and out (staged): same bits


ROUND_TRIPS = [
    (2, dict()),                             # config 2 at full size
    (3, dict(time_steps=8192)),              # wave, two slabs
    (5, dict(batch=8)),                      # 8 of config 5's problems at full size
    (4, dict()),                             # config 4 at full size: 65536 x 65536 (103 GB of buffers)
]
RT_IDS = ["cfg2-full", "cfg3-8192", "cfg5-8-full", "cfg4-full"]


@pytest.mark.parametrize("cid,kw", ROUND_TRIPS, ids=RT_IDS)
def test_round_trip_solve_of_apply(ft, cid, kw, record_property):
    """solve_fast(A x) = x for a smooth field x (the config's separable mode field): forward
    error max |u - x| / max |x| <= 1e-10.  A x in the difference form is accurate to
    ~eps b |x_(i+1) - x_i|, so the recovered x tests the whole solve -- every slab's leaf, the
    slab coupling, the in-leaf windows and all product levels -- at full width and length."""
    import torch

    torch.cuda.empty_cache()
    w = W.config(cid, **kw)
    plan = ft.Plan(w.specs)
    x = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    plan.assemble_rhs_modes(x, w.a, w.k, w.p, w.trig, None, None)   # used as the field x, not as a RHS
    R = plan.apply(x)
    U, rep = plan.solve_fast(R)
    err = ((U - x).abs().max() / x.abs().max()).item()
    record_property("solve_of_apply_rel_err", err)
    print(f"cfg{cid} {tuple(plan.shape)}: max|solve(A x) - x| / max|x| = {err:.3e} ({rep.kernel_launches} launches)")
    del U, R, x, plan
    torch.cuda.empty_cache()
    assert err <= 1e-10


@pytest.mark.parametrize("cid,kw", ROUND_TRIPS, ids=RT_IDS)
def test_round_trip_residual(ft, cid, kw, record_property):
    """A . solve_fast(R) - R, as the normwise backward error
    eta = max |A u - R| / (||A||_inf max |u| + max |R|)  (R: the config's own forcing).
    The residual relative to R alone is bounded below by eps ||A|| |u| / |R| (~4e-8 on config 4,
    ||A|| = 4 / h^2 = 1.7e10: one ulp of u times the stencil), so it is reported, not asserted."""
    import torch

    torch.cuda.empty_cache()
    w = W.config(cid, **kw)
    plan = ft.Plan(w.specs)
    R = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    plan.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig, w.u0amp, w.phiamp)
    U, _ = plan.solve_fast(R)
    work = torch.empty_like(R)
    res, rmax = plan.residual(R, U, work)
    umax = U.abs().max().item()
    s0 = w.specs[0]
    stencil = {3: 2.0 / s0.h() ** 2, 2: 1.0 / s0.h()}.get(int(s0.scheme), 0.0)
    anorm = max(np.abs(plan.column(b)).sum() for b in range(len(w.specs))) + stencil
    eta = res / (anorm * umax + rmax)
    record_property("backward_error", eta)
    record_property("residual_rel_rhs", res / rmax)
    print(f"cfg{cid} {tuple(plan.shape)}: eta = {eta:.3e}, max|A u - R| / max|R| = {res / rmax:.3e}")
    del work, U, R, plan
    torch.cuda.empty_cache()
    assert eta <= 1e-14


def test_apply_rejects_unsupported(ft):
    import torch

    w = W.transport(0.45, 256, 65, 0.6)
    plan = ft.Plan(w.specs)
    x = torch.zeros(plan.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ft.InvalidArgument):
        plan.apply(x)
    w = W.config(2, time_steps=64, cells=17)
    plan = ft.Plan(w.specs)
    x = torch.zeros(plan.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ft.InvalidArgument):
        plan.apply(x, x)


@pytest.mark.parametrize("cid,kw", [(1, dict(time_steps=300)), (2, dict(time_steps=200, cells=33)),
                                    (3, dict(time_steps=200, cells=700)), (4, dict(time_steps=128, cells=1100))],
                         ids=["ode", "diffusion", "wave-2-slabs", "diffusion-3-slabs"])
def test_homogeneous_problem_gives_zero(ft, cid, kw):
    """Zero right-hand side -> exactly zero solution on both paths (reference
    test_schemes.cpp:268-272 'homogeneous problems give 0')."""
    import torch

    w = W.config(cid, **kw)
    plan = ft.Plan(w.specs)
    R = torch.zeros(plan.shape, dtype=torch.float64, device="cuda")
    Uf, _ = plan.solve_fast(R)
    Ud, _ = plan.solve_direct(R)
    assert torch.count_nonzero(Uf).item() == 0 and torch.count_nonzero(Ud).item() == 0


@pytest.mark.parametrize("scheme,cells,steps", [(3, 9, 16), (3, 17, 12), (2, 9, 16)],
                         ids=["diffusion-8x16", "diffusion-16x12", "wave-8x16"])
def test_operator_entries_equal_time_marching_matrix(ft, scheme, cells, steps):
    """The reference's permutation-equivalence criterion (test_schemes.cpp:226-257, acceptance
    criterion 7, M, N <= 16): the node-major block operator equals, entry by entry, the stacked
    time-marching matrix -- row (i, n) holds col[n - k] at (i, k), k <= n, and the stencil at the
    neighbours (i +- 1, n).  The operator's columns come from ft_apply on unit vectors (all lags
    are in-leaf at N <= 16: single products, exact)."""
    import torch

    from paper_1710_11593_b200 import ProblemSpec, SchemeId

    s = ProblemSpec(SchemeId(scheme), 0.6 if scheme == 3 else 1.5, steps, cells, 1.0, 1.0)
    plan = ft.Plan([s])
    M, N = plan.shape
    col = plan.column(0)
    h = s.h()
    A = np.zeros((M * N, M * N))
    for i in range(M):
        for n in range(N):
            r = i * N + n
            for k in range(n + 1):
                A[r, i * N + k] = col[n - k]
            if scheme == 3:
                if i > 0:
                    A[r, (i - 1) * N + n] = -1.0 / (h * h)
                if i + 1 < M:
                    A[r, (i + 1) * N + n] = -1.0 / (h * h)
            elif i > 0:
                A[r, (i - 1) * N + n] = -1.0 / h
    E = torch.eye(M * N, dtype=torch.float64, device="cuda")
    got = np.empty_like(A)
    for c in range(M * N):
        got[:, c] = plan.apply(E[c].reshape(M, N).contiguous()).reshape(-1).cpu().numpy()
    # the stencil is applied in the difference form (d - 2b) x - b ((xl - x) + (xr - x)): on a unit
    # vector the diagonal entry is re-formed as (d - 2b) + 2b (or (d - s) + s), exact up to one rounding
    off = ~np.eye(M * N, dtype=bool)
    assert np.array_equal(got[off], A[off])
    d = np.abs(np.diag(got) - np.diag(A)) / np.abs(np.diag(A))
    assert d.max() <= 2.3e-16


def test_report_residual_option(ft):
    """ft_report::residual: 0 by default (direct method, as the reference's Direct path), the measured
    max |A u - rhs| / max |rhs| with FT_OPT_REPORT_RESIDUAL (SolveReport::residual, schemes.hpp:58-63)."""
    import torch

    w = W.config(2, time_steps=2048)
    plain = ft.Plan(w.specs)
    R = torch.empty(plain.shape, dtype=torch.float64, device="cuda")
    plain.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig, w.u0amp, w.phiamp)
    _, rep0 = plain.solve_fast(R)
    assert rep0.residual == 0.0
    plan = ft.Plan(w.specs, report_residual=True)
    Uf, repf = plan.solve_fast(R)
    Ud, repd = plan.solve_direct(R)
    res, rmax = plan.residual(R, Uf)
    assert 0.0 < repf.residual <= 1e-10 and repf.residual == res / rmax
    assert 0.0 < repd.residual <= 1e-10
