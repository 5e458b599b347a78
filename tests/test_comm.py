"""CPU tests of the sharding host layer: shard geometry, the
loopback communicator objects, and the torch.distributed all-gather backend
driven through its C function pointer by two gloo ranks (world_size 2)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2404_16370_b200 import comm as CM
from paper_2404_16370_b200.abi import ALLGATHER_FN, ALLTOALLV_FN


def test_shard_range_contiguous_and_aligned():
    n = 4096 * 8
    spans = [CM.shard_range(n, r, 4) for r in range(4)]
    assert spans == [(0, 8192), (8192, 8192), (16384, 8192), (24576, 8192)]
    assert CM.shard_range(4096, 0, 1) == (0, 4096)
    with pytest.raises(ValueError):
        CM.shard_range(4096 * 3, 0, 2)  # 6144 per shard is not chunk aligned
    with pytest.raises(ValueError):
        CM.shard_range(8192, 2, 2)


def test_loopback_comms_fill_rank_and_world():
    c = CM.LoopbackComms(3)
    assert [c[r].rank for r in range(3)] == [0, 1, 2]
    assert all(c[r].world == 3 and c[r].ctx for r in range(3))
    assert all(bool(c[r].allgather) and bool(c[r].alltoallv) for r in range(3))
    c.close()
    c.close()  # idempotent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tc = CM.TorchComm(device=False)
        assert (tc.struct.rank, tc.struct.world) == (rank, world)
        fn = C.cast(tc.struct.allgather, ALLGATHER_FN)  # call through the C function pointer
        for nbytes in (8, 96 * 5, 4096 * 8):
            send = (np.arange(nbytes, dtype=np.uint64) * 7 + rank * 1000003).astype(np.uint8)
            recv = np.zeros(nbytes * world, np.uint8)
            rc = fn(None, send.ctypes.data, recv.ctypes.data, nbytes, None)
            assert rc == 0, tc.error
            for r in range(world):
                exp = (np.arange(nbytes, dtype=np.uint64) * 7 + r * 1000003).astype(np.uint8)
                assert np.array_equal(recv[r * nbytes:(r + 1) * nbytes], exp)
        assert fn(None, None, None, 0, None) == 0  # empty all-gather is a no-op
        # alltoallv: rank r sends (r + 1) * (d + 1) * 3 bytes to rank d (one chunk empty)
        a2a = C.cast(tc.struct.alltoallv, ALLTOALLV_FN)
        size = lambda s, d: 0 if (s, d) == (1, 0) else (s + 1) * (d + 1) * 3
        sb = (C.c_uint64 * world)(*[size(rank, d) for d in range(world)])
        rb = (C.c_uint64 * world)(*[size(s, rank) for s in range(world)])
        send = np.concatenate([np.full(size(rank, d), 16 * rank + d, np.uint8) for d in range(world)])
        recv = np.zeros(sum(rb), np.uint8)
        assert a2a(None, send.ctypes.data, sb, recv.ctypes.data, rb, None) == 0, tc.error
        exp = np.concatenate([np.full(size(s, rank), 16 * s + rank, np.uint8) for s in range(world)])
        assert np.array_equal(recv, exp)
        out.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        out.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_torch_comm_gloo_allgather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}
