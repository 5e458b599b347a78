"""Native NCCL communicator (smcl_comm_nccl_create): a one-rank communicator on
the test GPU runs the engine-facing all-gather entry point on device buffers.
(Multi-rank behaviour of the exchange plan is covered by the loopback and
gloo tests; this pins the NCCL binding itself.)"""
import ctypes as C

import numpy as np
import pytest

from paper_2404_16370_b200.comm import NcclComm

pytestmark = pytest.mark.gpu


def test_nccl_comm_world1_allgather():
    import torch
    torch.cuda.set_device(0)
    comm = NcclComm(NcclComm.unique_id(), 0, 1)
    assert comm.struct.world == 1 and comm.struct.ctx
    src = torch.arange(1000, dtype=torch.int32, device="cuda")
    dst = torch.zeros(1000, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    rc = comm.struct.allgather(comm.struct.ctx, C.c_void_p(src.data_ptr()), C.c_void_p(dst.data_ptr()),
                               C.c_uint64(4000), C.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0
    assert np.array_equal(dst.cpu().numpy(), np.arange(1000))
    comm.close()


def test_nccl_comm_world1_alltoallv():
    """alltoallv = one group of ncclSend/ncclRecv (a self exchange at world 1)."""
    import torch
    torch.cuda.set_device(0)
    comm = NcclComm(NcclComm.unique_id(), 0, 1)
    assert comm.struct.alltoallv
    src = torch.arange(1000, dtype=torch.int32, device="cuda")
    dst = torch.zeros(1000, dtype=torch.int32, device="cuda")
    nb = (C.c_uint64 * 1)(4000)
    stream = torch.cuda.current_stream()
    rc = comm.struct.alltoallv(comm.struct.ctx, C.c_void_p(src.data_ptr()), nb, C.c_void_p(dst.data_ptr()), nb,
                               C.c_void_p(stream.cuda_stream))
    torch.cuda.synchronize()
    assert rc == 0 and np.array_equal(dst.cpu().numpy(), np.arange(1000))
    comm.close()
