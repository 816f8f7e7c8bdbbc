"""The reference-shaped entry points, used the way the reference's callers use
them: solve(spec, method) with std::function-style callbacks evaluated inside
the call (reference schemes.cpp:481-489, forcing at :401-408 / :300-306 /
:183-187, called from harness.cpp:154-170), and ft_assemble_rhs with callbacks.
The unmodified reference (oracle/_ref) runs on identical callback values."""
import math

import numpy as np
import pytest

from paper_1710_11593_b200 import SchemeId, SolveMethod
from paper_1710_11593_b200 import workloads as W

pytestmark = pytest.mark.gpu
PI = math.pi


def _specs(ft):
    f4 = lambda x, t: math.sin(PI * x) * (1.0 + t * t) + math.cos(3.0 * x) * t  # noqa: E731
    f3 = lambda x, t: math.sin(PI * x) * t * t + math.cos(PI * x)  # noqa: E731
    return {
        "diffusion": ft.ProblemSpec(SchemeId.Diffusion, 0.7, 300, 41, 1.0, 1.0, forcing=f4),
        "diffusion-u0": ft.ProblemSpec(SchemeId.Diffusion, 0.3, 257, 33, 1.0, 1.0, forcing=f4,
                                       initial_u0=lambda x: math.sin(PI * x)),
        "wave": ft.ProblemSpec(SchemeId.DiffusionWave, 1.5, 200, 33, 1.0, 1.0, forcing=f3,
                               initial_u0=lambda x: math.sin(PI * x), initial_phi=lambda x: 0.5 * math.sin(PI * x)),
        "transport": ft.ProblemSpec(SchemeId.Hyperbolic, 0.45, 128, 65, 1.0, 1.0, forcing=f4,
                                    initial_u0=lambda x: math.sin(PI * x)),
    }


def _grids(spec):
    """The callbacks sampled at the reference's evaluation points, with the same
    double expressions (so the reference's grid-lookup callbacks see the same values)."""
    h, tau, N = spec.h(), spec.tau(), spec.time_steps
    xs = [float(i) * h for i in range(1, spec.space_cells)]
    if spec.scheme == SchemeId.Hyperbolic:
        xs = [(float(i) - 0.5) * h for i in range(1, spec.space_cells)]
    ts = [(float(n) - 0.5) * tau if spec.scheme == SchemeId.DiffusionWave else float(n) * tau for n in range(1, N + 1)]
    F = np.array([[spec.forcing(x, t) for t in ts] for x in xs])
    u0 = phi = None
    if spec.initial_u0 is not None:
        r = range(0, spec.space_cells) if spec.scheme == SchemeId.Hyperbolic else range(1, spec.space_cells)
        u0 = np.array([spec.initial_u0(float(i) * h) for i in r])
    if spec.initial_phi is not None:
        phi = np.array([spec.initial_phi(float(i) * h) for i in range(1, spec.space_cells)])
    return F, u0, phi


@pytest.mark.parametrize("name", ["diffusion", "diffusion-u0", "wave", "transport"])
def test_solve_spec_callbacks_vs_reference(ft, oracle_mod, name):
    if oracle_mod.rlib() is None:
        pytest.fail("oracle/_ref (the unmodified reference) is not built")
    spec = _specs(ft)[name]
    F, u0, phi = _grids(spec)
    ref, _, _ = oracle_mod.ref_solve(spec, "direct", F, u0, phi)
    fast = ft.solve(spec, SolveMethod.Fast)
    direct = ft.solve(spec, SolveMethod.Direct)
    assert fast.report.method == "fast" and direct.report.method == "direct"
    assert fast.report.iterations == 0 and fast.report.kernel_launches > 0
    assert fast.grid.values.shape == ((spec.space_cells - 1) * spec.time_steps,)
    Uf = fast.grid.values.reshape(ref.shape)
    Ud = direct.grid.values.reshape(ref.shape)
    assert oracle_mod.relerr(Uf, ref) <= 1e-10
    if u0 is None or spec.scheme == SchemeId.Hyperbolic:
        assert np.array_equal(Ud, ref)  # same RHS, same summation order, no FMA
    else:
        assert oracle_mod.relerr(Ud, ref) <= 1e-14
    assert fast.grid.at(3, 7) == Uf[2, 6]


@pytest.mark.parametrize("name", ["diffusion-u0", "wave", "transport"])
def test_assemble_rhs_callbacks_equals_grid_form(ft, name):
    spec = _specs(ft)[name]
    F, u0, phi = _grids(spec)
    plan = ft.Plan(spec)
    R1 = plan.assemble_rhs(spec.forcing, spec.initial_u0, spec.initial_phi)
    R2 = plan.assemble_rhs_grid(F, u0, phi)
    assert np.array_equal(R1, R2)


def test_assemble_rhs_callbacks_vs_reference_golden(ft):
    """ft_assemble_rhs with grid-lookup callbacks (as the reference shim feeds the
    reference) reproduces the reference's assemble_scheme4 RHS bitwise."""
    from pathlib import Path

    g = np.load(Path(__file__).resolve().parent / "golden" / "golden.npz")
    w = W.config(2, time_steps=128, cells=17)
    s = w.specs[0]
    F, u0 = g["cfg2_m16_n128_F"], g["cfg2_m16_n128_u0"]
    h, tau = s.h(), s.tau()
    plan = ft.Plan(w.specs)
    R = plan.assemble_rhs(lambda x, t: float(F[round(x / h) - 1, round(t / tau) - 1]),
                          lambda x: float(u0[round(x / h) - 1]))
    assert np.array_equal(R, g["cfg2_m16_n128_rhs"])


def test_buffer_validation(ft):
    """Wrong dtype / size / layout buffers are rejected before they reach the C ABI."""
    import torch

    w = W.config(2, time_steps=64, cells=17)
    plan = ft.Plan(w.specs)
    good = torch.zeros(plan.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ft.InvalidArgument):
        plan.solve_fast(good.float())
    with pytest.raises(ft.InvalidArgument):
        plan.solve_fast(good[:, :32].contiguous(), torch.empty_like(good))
    with pytest.raises(ft.InvalidArgument):
        plan.solve_fast(good.t())
    with pytest.raises(ft.InvalidArgument):
        plan.solve_fast_modes(good, w.a[:, :2], w.k, w.p, w.trig)


def test_concurrent_batched_plans_on_distinct_streams(ft):
    """Two batched plans (per-problem leaf weights in the device's constant bank)
    solving concurrently from two host threads on two streams give exactly their
    serial results (the bank is handed over in stream order, ft_destroy forgets it)."""
    import threading

    import torch

    wa = W.config(5, time_steps=2048, batch=3)
    wb = W.config(5, time_steps=2048, batch=5)
    wb.specs = [ft.ProblemSpec(s.scheme, 0.95 - s.gamma, s.time_steps, s.space_cells, s.time_length,
                               s.space_length) for s in wb.specs]
    out = {}
    for name, w in (("a", wa), ("b", wb)):
        plan = ft.Plan(w.specs)
        R = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
        plan.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig, w.u0amp, w.phiamp)
        U, _ = plan.solve_fast(R, torch.empty_like(R))
        out[name] = (plan, R, U.clone())
    errs = []

    def worker(name):
        plan, R, ref = out[name]
        st = torch.cuda.Stream()
        plan.set_stream(st.cuda_stream)
        U = torch.empty_like(R)
        for _ in range(6):
            plan.solve_fast(R, U)
            if not torch.equal(U, ref):
                errs.append(name)

    ths = [threading.Thread(target=worker, args=(n,)) for n in ("a", "b")]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
