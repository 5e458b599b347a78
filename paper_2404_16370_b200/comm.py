"""Collective backends for sharded engines.

A sharded engine (``smcl_create_sharded``) owns the particles with global
indices ``[rank*N/world, (rank+1)*N/world)`` and calls an all-gather on its
own CUDA stream (plus, with ``reorder_particles``, an alltoallv of the
particle records that change shard) at the exchange points of
``FilterEngine::step`` (filter.cpp:118-213): LSH keys before the global sort,
poses/steps before each SVGD iteration, per-chunk partial sums and argmax
partials of the posterior reductions, the per-round probabilities of the
smoothing passes and the representative pose. Everything else is shard-local.

Backends:

* ``LoopbackComms`` — in-process, ``world`` engines driven by ``world`` host
  threads (one device or several); implemented in C (engine.cu).
* ``NcclComm`` — native NCCL (``smcl_comm_nccl_create``): the engine calls
  ``ncclAllGather`` / grouped ``ncclSend``+``ncclRecv`` on its own stream,
  no Python on the data path. The
  128-byte unique id travels over any host channel (``NcclComm.from_torch``
  uses the torch.distributed group bench.py already has).
* ``TorchComm`` — ``torch.distributed`` over NCCL (device buffers, one process
  per GPU), gloo on host buffers (the CPU tests of this layer), or gloo
  host-staged (``staged=True``: the engine's device buffers are copied to the
  host around a gloo collective after its stream drains, so several
  processes can drive sharded engines on one GPU with no kernel ever waiting
  on another process — the two-process GPU test).

torch is plumbing here: it is imported lazily and only by ``TorchComm``.
"""
import ctypes as C

from . import _lib
from .abi import ALLGATHER_FN, ALLTOALLV_FN, SmclComm

SHARD_ALIGN = 4096  # reduce.hpp chunk: no posterior reduction chunk straddles two shards


def shard_range(n_total, rank, world):
    """(gbase, n_local) of ``rank`` for ``n_total`` particles over ``world`` shards."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    if n_total % world or (n_total // world) % SHARD_ALIGN:
        raise ValueError(f"N={n_total} over {world} shards: N/world must be a multiple of {SHARD_ALIGN}")
    n_local = n_total // world
    return rank * n_local, n_local


class LoopbackComms:
    """``world`` in-process communicators (smcl_comm_loopback_create)."""

    def __init__(self, world):
        self.world = world
        self.structs = (SmclComm * world)()
        _lib.check(_lib.lib().smcl_comm_loopback_create(world, self.structs))

    def __getitem__(self, rank):
        return self.structs[rank]

    def close(self):
        if self.structs is not None:
            _lib.lib().smcl_comm_loopback_destroy(self.structs)
            self.structs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NcclComm:
    """Native NCCL communicator for one rank (libnccl.so.2, NVLink/NVSwitch)."""

    @staticmethod
    def unique_id():
        buf = (C.c_uint8 * 128)()
        _lib.check(_lib.lib().smcl_nccl_get_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid, rank, world):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self.struct = SmclComm()
        _lib.check(_lib.lib().smcl_comm_nccl_create(buf, rank, world, C.byref(self.struct)))
        self.rank, self.world = rank, world

    @classmethod
    def from_torch(cls, group=None):
        """Rank 0 makes the id, torch.distributed broadcasts it, every rank joins
        (call with this rank's CUDA device current)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], rank, world)

    def close(self):
        if getattr(self, "struct", None) is not None and self.struct.ctx:
            _lib.lib().smcl_comm_nccl_destroy(C.byref(self.struct))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DeviceBytes:
    """Zero-copy uint8 view of raw device memory for torch.as_tensor."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


class TorchComm:
    """smcl_comm over a torch.distributed process group.

    ``device=True`` (NCCL): send/recv are device pointers of the engine's GPU
    and the all-gather is enqueued on the engine's stream (ExternalStream), so
    it is ordered after the engine's producers and before its consumers.
    ``device=False`` (gloo): send/recv are host pointers.
    ``staged=True`` (gloo): send/recv are device pointers; the engine stream is
    drained, the bytes go through host memory and are back on the device
    before the call returns.
    """

    def __init__(self, group=None, device=True, staged=False):
        import torch.distributed as dist
        self.group = group
        self.device = device and not staged
        self.staged = staged
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.error = None
        self._fn = ALLGATHER_FN(self._allgather)  # keep the trampolines alive
        self._fn_a2a = ALLTOALLV_FN(self._alltoallv)
        self.struct = SmclComm(None, self.rank, self.world, self._fn, self._fn_a2a)

    def _allgather(self, ctx, send, recv, nbytes, stream):
        try:
            import torch
            import torch.distributed as dist
            nbytes = int(nbytes)
            if nbytes == 0:
                return 0
            if self.staged:
                dev = torch.device("cuda", torch.cuda.current_device())
                torch.cuda.ExternalStream(int(stream or 0), device=dev).synchronize()
                s = torch.as_tensor(_DeviceBytes(send, nbytes), device=dev).cpu()
                parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(parts, s, group=self.group)
                r = torch.as_tensor(_DeviceBytes(recv, nbytes * self.world), device=dev)
                r.copy_(torch.cat(parts))
                torch.cuda.synchronize(dev)
            elif self.device:
                dev = torch.device("cuda", torch.cuda.current_device())
                s = torch.as_tensor(_DeviceBytes(send, nbytes), device=dev)
                r = torch.as_tensor(_DeviceBytes(recv, nbytes * self.world), device=dev)
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0), device=dev)):
                    dist.all_gather_into_tensor(r, s, group=self.group)
            else:
                s = torch.frombuffer((C.c_uint8 * nbytes).from_address(send), dtype=torch.uint8)
                r = torch.frombuffer((C.c_uint8 * (nbytes * self.world)).from_address(recv), dtype=torch.uint8)
                dist.all_gather(list(r.split(nbytes)), s.clone(), group=self.group)
            return 0
        except Exception as e:  # surfaced by the engine as an SMCL error
            self.error = e
            return 1

    def _alltoallv(self, ctx, send, send_bytes, recv, recv_bytes, stream):
        try:
            import torch
            import torch.distributed as dist
            sb = [int(send_bytes[i]) for i in range(self.world)]
            rb = [int(recv_bytes[i]) for i in range(self.world)]
            ns, nr = sum(sb), sum(rb)
            if self.staged:
                dev = torch.device("cuda", torch.cuda.current_device())
                torch.cuda.ExternalStream(int(stream or 0), device=dev).synchronize()
                s = (torch.as_tensor(_DeviceBytes(send, ns), device=dev).cpu() if ns
                     else torch.empty(0, dtype=torch.uint8))
                r = torch.empty(nr, dtype=torch.uint8)
                dist.all_to_all_single(r, s, output_split_sizes=rb, input_split_sizes=sb, group=self.group)
                if nr:
                    torch.as_tensor(_DeviceBytes(recv, nr), device=dev).copy_(r)
                    torch.cuda.synchronize(dev)
            elif self.device:
                dev = torch.device("cuda", torch.cuda.current_device())
                s = torch.as_tensor(_DeviceBytes(send, ns), device=dev) if ns else torch.empty(0, dtype=torch.uint8,
                                                                                                device=dev)
                r = torch.as_tensor(_DeviceBytes(recv, nr), device=dev) if nr else torch.empty(0, dtype=torch.uint8,
                                                                                                device=dev)
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0), device=dev)):
                    dist.all_to_all_single(r, s, output_split_sizes=rb, input_split_sizes=sb, group=self.group)
            else:
                s = (torch.frombuffer((C.c_uint8 * ns).from_address(send), dtype=torch.uint8).clone() if ns
                     else torch.empty(0, dtype=torch.uint8))
                r = torch.empty(nr, dtype=torch.uint8)
                dist.all_to_all_single(r, s, output_split_sizes=rb, input_split_sizes=sb, group=self.group)
                if nr:
                    C.memmove(recv, r.data_ptr(), nr)
            return 0
        except Exception as e:
            self.error = e
            return 1
