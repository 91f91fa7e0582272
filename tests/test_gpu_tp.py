"""lutgemm_tp_linear on one GPU (world size 1 NCCL communicator): every mode against
the fp64 oracle (north_star tolerances), and the row modes also bitwise equal to the
single-GPU product (the m-split keeps each row's fixed-order reduction)."""
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
from tests._helpers import assert_parity
from workloads import gen_bcq, gen_x

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def comm():
    import torch.distributed as dist

    import paper_2206_09557_b200 as L
    if not dist.is_initialized():
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    c = L.TPComm(0, 1)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("b", [1, 2, 3, 8])
def test_tp_world1_modes(comm, b):
    import paper_2206_09557_b200 as L
    m, n, q, g = 1024, 2048, 3, 128
    d = gen_bcq(41, m, n, q, g, offset=True)
    w = L.lutgemm_pack_bcq(dev(d["planes"].view(np.int32)), dev(d["alpha"]), dev(d["offset"]), n, g)
    X = dev(gen_x(41, b, n))
    ref_dev = L.lutgemm_gemm_batched(w, X) if b > 1 else L.lutgemm_gemv(w, X[0])[None]
    ref = O.bcq_gemv(d["planes"], d["alpha"], d["offset"], gen_x(41, b, n), n, g)
    for mode in (L.TP_ROWS_LOCAL, L.TP_ROWS_ALLGATHER, L.TP_COLS_ALLREDUCE):
        ws = L.make_workspace(comm.workspace_bytes(mode, m, n, b), "cuda")
        y = torch.empty((b, m), dtype=torch.float16, device="cuda")
        comm.linear(mode, w, X if b > 1 else X[0], y, ws)
        torch.cuda.synchronize()
        assert_parity(y.float().cpu().numpy(), ref, ("tp", mode, b))
        if mode != L.TP_COLS_ALLREDUCE:
            assert torch.equal(y, ref_dev), mode
