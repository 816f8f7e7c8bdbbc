"""Multi-GPU execution of the fast solver.

* Independent problems (config 5): `shard_problems` splits a batch over ranks;
  each rank builds an ordinary batched plan -- no communication.
* One wide problem (config 4): `ShardedPlan` holds rank r's contiguous slab
  range (ft_setup_partitioned).  History products are node-local; the leaf
  all-gathers its slabs' scan carries once per leaf through an exchange hook
  registered with ft_set_exchange.  `torch_exchange` implements the hook with
  torch.distributed (NCCL on GPUs; gloo for CPU tests) on the plan's stream.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Sequence, Tuple

import torch

from . import EXCHANGE_FN, Plan, _check, lib


def partition_range(count: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [begin, end) of `count` items for `rank` (balanced)."""
    base, extra = divmod(count, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def shard_problems(specs: Sequence, rank: int, world: int) -> List:
    b, e = partition_range(len(specs), rank, world)
    return list(specs[b:e])


def slab_partition(nodes: int, world: int, slab: int = 512) -> List[Tuple[int, int]]:
    """Node ranges of a slab-aligned partition (what ft_setup_partitioned uses)."""
    slabs = -(-nodes // slab)
    if slabs % world:
        raise ValueError(f"{slabs} slabs do not divide over {world} ranks")
    per = slabs // world
    return [(r * per * slab, min(nodes, (r + 1) * per * slab)) for r in range(world)]


def torch_exchange(send: torch.Tensor, recv: torch.Tensor, stream=None, group=None) -> Callable[[int], None]:
    """All-gather `send` (count doubles) from every rank into `recv` (rank-major)."""
    import torch.distributed as dist

    backend = dist.get_backend(group)

    def run(count: int) -> None:
        world = dist.get_world_size(group)
        if send.numel() != count or recv.numel() != count * world:
            raise ValueError(f"exchange: {count} doubles per rank, buffers {send.numel()} / {recv.numel()}")
        ctx = torch.cuda.stream(stream) if (stream is not None and send.is_cuda) else _null()
        with ctx:
            if backend == "nccl":
                dist.all_gather_into_tensor(recv, send, group=group)
            elif send.is_cuda:
                # gloo moves host tensors: stage through the host (the copy waits for this
                # rank's phase-1 kernel on `stream`; the result lands before the correction)
                host = send.cpu()
                parts = [torch.empty_like(host) for _ in range(world)]
                dist.all_gather(parts, host, group=group)
                recv.copy_(torch.cat(parts))
            else:
                parts = list(recv.view(world, -1).unbind(0))
                dist.all_gather(parts, send, group=group)

    return run


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class ShardedPlan(Plan):
    """Rank `rank` of `world`'s share of one wide problem.  `exchange(count)` is
    called once per leaf and must all-gather `count` doubles per rank from
    `self.send` into `self.recv` on `self.stream`."""

    def __init__(self, spec, rank: int, world: int, exchange_factory=None, device: int = -1, p2p: bool = False,
                 native_nccl: bool = False, **kw):
        super().__init__(spec, partition=(rank, world), device=device, **kw)
        self.rank, self.world = rank, world
        P_local, L = int(self.info.slabs_local), int(self.info.leaf)
        dev = torch.device("cuda", torch.cuda.current_device() if device < 0 else device)
        self.send = torch.zeros(P_local * L * 2, dtype=torch.float64, device=dev)
        self.recv = torch.zeros(world * P_local * L * 2, dtype=torch.float64, device=dev)
        self.stream = torch.cuda.Stream(device=dev)
        self.set_stream(self.stream.cuda_stream)
        factory = exchange_factory or (lambda send, recv, stream: torch_exchange(send, recv, stream))
        self._exchange = factory(self.send, self.recv, self.stream)

        def hook(_user, count, _stream):
            try:
                self._exchange(int(count))
                return 0
            except Exception:  # noqa: BLE001 -- reported through the ABI return code
                import traceback

                traceback.print_exc()
                return 1

        self._hook = EXCHANGE_FN(hook)  # keep alive
        _check(lib().ft_set_exchange(self._h, self._hook, None, self.send.data_ptr(), self.recv.data_ptr()))
        if p2p:
            self.connect_peers()
        elif native_nccl:
            self.bind_nccl()

    def bind_nccl(self, group=None) -> None:
        """The carry all-gather as ncclAllGather issued by the library on the plan's stream
        (ft_nccl_init): rank 0's unique id is broadcast over torch.distributed (any backend),
        every rank joins the solver's own communicator; solves then replay as one CUDA graph."""
        import torch.distributed as dist

        from . import nccl_unique_id

        box = [nccl_unique_id() if self.rank == 0 else None]
        if self.world > 1:
            dist.broadcast_object_list(box, src=0, group=group)
        self.nccl_init(box[0], self.rank, self.world)

    def connect_peers(self, group=None) -> None:
        """Switch to the in-kernel exchange over NVLink peer memory: all-gather the
        ranks' CUDA IPC handles (any torch.distributed backend) and map them."""
        import torch.distributed as dist

        h = (C.c_ubyte * 64)()
        _check(lib().ft_p2p_handle(self._h, h))
        handles = [None] * self.world
        dist.all_gather_object(handles, bytes(h), group=group)
        blob = b"".join(handles)
        buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(lib().ft_p2p_connect(self._h, buf))
