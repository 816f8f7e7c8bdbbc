"""The carry all-gather as ncclAllGather issued by the library (ft_nccl_init), captured with the
rest of the solve into one CUDA graph.  Every GPU tier of this run has one GPU, so the path is
exercised with a one-rank communicator: the same two-kernel leaf (phase 1 / all-gather /
correction), the same buffers and the same graph capture as on N ranks; the slab partition itself
is covered across 2 and 4 processes by tests/test_parallel.py (gloo exchange)."""
import pytest

from paper_1710_11593_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid,kw", [(4, dict(time_steps=1024, cells=2049)),      # 5 slabs, ragged last
                                    (3, dict(time_steps=512, cells=1025))],     # wave scheme, 2 slabs
                         ids=["diffusion-5-slabs", "wave-2-slabs"])
def test_native_nccl_exchange_one_rank(ft, cid, kw):
    import torch

    w = W.config(cid, **kw)
    plan = ft.Plan(w.specs)
    R = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    plan.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig, w.u0amp, w.phiamp)
    U0, rep0 = plan.solve_fast(R)
    try:
        uid = ft.nccl_unique_id()
    except ft.FractimeError as e:
        pytest.skip(f"NCCL not loadable here: {e}")
    plan2 = ft.Plan(w.specs)
    plan2.nccl_init(uid, 0, 1)
    U1, rep1 = plan2.solve_fast(R)
    U2, rep2 = plan2.solve_fast(R)   # graph replay with the collectives inside
    assert torch.equal(U2, U1)
    if cid == 3:
        # Scheme 3 plans of <= 4 slabs default to the chained-slab leaf (exact, no correction phase):
        # same solution as the phase-1 / all-gather / correction path to rounding, not to the bit
        err = ((U1 - U0).abs().max() / U0.abs().max()).item()
        assert err <= 1e-12, err
    else:
        assert torch.equal(U1, U0)
    leaves = (plan.N + 31) // 32
    # two kernels per leaf (the collective between them) instead of one cooperative kernel
    assert rep1.kernel_launches >= 2 * leaves and rep1.kernel_launches == rep2.kernel_launches
    assert rep1.kernel_launches > rep0.kernel_launches


def test_nccl_init_rejects_bad_arguments(ft):
    w = W.config(2, time_steps=64, cells=17)      # single slab: nothing to exchange
    plan = ft.Plan(w.specs)
    with pytest.raises(ft.InvalidArgument):
        plan.nccl_init(bytes(128), 0, 1)
    w = W.config(4, time_steps=64, cells=1025)
    plan = ft.Plan(w.specs)
    with pytest.raises(ft.InvalidArgument):
        plan.nccl_init(bytes(128), 1, 2)          # not this plan's partition


def test_fast_solve_is_bitwise_reproducible(ft):
    """Repeated solves (CUDA-graph replays) and a second plan give identical bits: every output
    is written by exactly one task in a fixed summation order -- including the split levels,
    whose fold / branch / combine tasks are handed out by a dynamic queue (n = 32768, 65536)."""
    import torch

    w = W.config(4, cells=1537)                      # 3 slabs, full N = 65536: every level incl. split K = 8, 16
    plan = ft.Plan(w.specs)
    R = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    plan.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig, w.u0amp, w.phiamp)
    U1, _ = plan.solve_fast(R)
    U2, _ = plan.solve_fast(R, torch.empty_like(R))
    plan2 = ft.Plan(w.specs)
    U3, _ = plan2.solve_fast(R)
    assert torch.equal(U1, U2) and torch.equal(U1, U3)
