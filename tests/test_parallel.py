"""Multi-rank paths.

CPU (gloo, world_size 2): the partition arithmetic and the per-leaf carry
exchange hook (torch_exchange) that ShardedPlan registers with the C ABI.
GPU (1 device): two ranks of a partitioned config-4-shaped problem run as two
host threads with their own plans/streams and an in-process exchange; the
stitched solution must be bitwise equal to the single-plan solve and within
1e-10 of the oracle.
"""
import os
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1710_11593_b200 import parallel as par
from paper_1710_11593_b200 import workloads as W


def test_partitions():
    for n, w in [(65536, 1), (65536, 2), (65536, 8), (4096, 8), (3000, 2)]:
        try:
            ranges = par.slab_partition(n, w)
        except ValueError:
            assert (-(-n // 512)) % w != 0
            continue
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        assert all(r[0] % 512 == 0 for r in ranges)
    for count, world in [(64, 8), (64, 3), (5, 8)]:
        got = [par.partition_range(count, r, world) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == count
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        assert max(e - b for b, e in got) - min(e - b for b, e in got) <= 1
    specs = W.config(5).specs
    assert sum(len(par.shard_problems(specs, r, 8)) for r in range(8)) == 64


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        count = 6
        send = torch.arange(count, dtype=torch.float64) + 100.0 * rank
        recv = torch.zeros(count * world, dtype=torch.float64)
        ex = par.torch_exchange(send, recv)
        for leaf in range(3):  # repeated per-leaf exchanges reuse the buffers
            send += 1.0
            ex(count)
            exp = torch.cat([torch.arange(count, dtype=torch.float64) + 100.0 * r + leaf + 1 for r in range(world)])
            assert torch.equal(recv, exp), (rank, leaf, recv)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


class _LocalExchange:
    """In-process all-gather between rank threads sharing one GPU."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.shared = None
        self.lock = threading.Lock()

    def factory(self, rank):
        def make(send, recv, stream):
            def run(count):
                with self.lock:
                    if self.shared is None:
                        self.shared = torch.zeros(count * self.world, dtype=torch.float64, device=send.device)
                stream.synchronize()  # this rank's phase 1 is done
                self.shared[rank * count:(rank + 1) * count].copy_(send)
                torch.cuda.synchronize()
                self.barrier.wait()
                with torch.cuda.stream(stream):
                    recv.copy_(self.shared)
                stream.synchronize()
                self.barrier.wait()  # nobody overwrites `shared` before everyone copied

            return run

        return make


@pytest.mark.gpu
@pytest.mark.parametrize("world,cells,steps,scheme", [(2, 4097, 200, 4), (4, 4097, 96, 4), (2, 65537, 64, 4),
                                                      (2, 2049, 128, 2), (4, 2049, 70, 2)])
def test_sharded_plan_matches_single(ft, oracle_mod, world, cells, steps, scheme):
    """scheme 4: config 4 shapes; scheme 2: transport (stencil history across the rank boundary)."""
    w = W.config(4, time_steps=steps, cells=cells) if scheme == 4 else W.transport(0.4, steps, cells, 1.0)
    F = oracle_mod.forcing_grid(w)
    u0 = oracle_mod.initial_grid(w, w.u0amp)
    single = ft.Plan(w.specs)
    R = single.assemble_rhs_grid(F, u0)
    U1, _ = single.solve_fast(R)
    ex = _LocalExchange(world)
    plans = [par.ShardedPlan(w.specs[0], r, world, exchange_factory=ex.factory(r)) for r in range(world)]
    outs = [None] * world
    errs = []

    def run(r):
        try:
            p = plans[r]
            b = p.node_begin
            Rl = np.ascontiguousarray(R[b:b + p.nodes])
            outs[r], _ = p.solve_fast(Rl)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ths = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    assert not errs, errs
    U = np.vstack(outs)
    assert np.array_equal(U, U1)
    if cells <= 4097:
        assert oracle_mod.relerr(U, oracle_mod.direct(w, F, u0)) <= 1e-10


def _sharded_worker(rank, world, port, cells, steps, q):
    """One rank of a slab-partitioned config-4-shaped solve in its own process (own CUDA
    context on the shared GPU), the default ShardedPlan exchange (torch_exchange over
    gloo: the per-leaf carry all-gather is host-synchronous, so no kernel waits on the
    other process)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        w = W.config(4, time_steps=steps, cells=cells)
        p = par.ShardedPlan(w.specs[0], rank, world)
        R = torch.empty(p.shape, dtype=torch.float64, device="cuda")
        p.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig)  # this rank's rows of the device RHS
        U, rep = p.solve_fast(R, torch.empty_like(R))
        q.put((rank, p.node_begin, U.cpu().numpy(), int(rep.kernel_launches)))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, -1, traceback.format_exc(), 0))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,cells,steps", [(2, 4097, 300), (4, 8193, 160)])
def test_sharded_plan_two_processes_gloo(ft, world, cells, steps):
    """ShardedPlan across `world` processes through torch.distributed (gloo): the
    stitched solution is bitwise equal to the single-plan solve."""
    import paper_1710_11593_b200 as ftm

    w = W.config(4, time_steps=steps, cells=cells)
    single = ftm.Plan(w.specs)
    R = torch.empty(single.shape, dtype=torch.float64, device="cuda")
    single.assemble_rhs_modes(R, w.a, w.k, w.p, w.trig)
    U1, _ = single.solve_fast(R, torch.empty_like(R))
    U1 = U1.cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, cells, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for rank, begin, U, _ in res:
        assert begin >= 0, U
    U = np.vstack([r[2] for r in res])
    assert [r[1] for r in res] == sorted(r[1] for r in res)
    assert np.array_equal(U, U1)
