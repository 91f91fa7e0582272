"""GPU parity for SURVEY 8(b)'s full shape contract: n % 8 == 0, g % 8 == 0, g | n (g is "an
arbitrary number of weights"), beyond the power-of-two groups of the BASELINE configs.

Group classes of the native layout (layout.cuh): groups straddling a 1024-column LUT slice
(g = 96, 384, 640, 1536), chunk groups that split a 32-column lane (g % 32 != 0: 8, 16, 24, 40, 72),
and n % 32 != 0 (a partial last lane, x staged as zero past n).  Every product is checked against
the fp64 oracle (oracle.bcq_gemv, which is written for any g and n) at the north_star tolerances,
for b = 1 (GEMV), b <= 4 and b > 4, with and without the offset term, and through the fused P2P
epilogue at world 1."""
import numpy as np
import pytest
import torch

import oracle as O
from tests._helpers import assert_parity
from workloads import gen_bcq, gen_uniform, gen_x

pytestmark = pytest.mark.gpu

SHAPES = [  # (m, n, q, g): the class each exercises
    (1000, 4800, 3, 96),     # straddling groups (1024 / 96 not whole)
    (777, 4608, 2, 384),     # straddling
    (513, 3200, 4, 640),     # straddling, several per slice boundary
    (300, 4608, 3, 1536),    # g > 1024, not a multiple: two groups in some slices
    (1029, 4104, 3, 24),     # chunk groups, n % 32 == 8
    (640, 1000, 2, 8),       # the smallest group, n % 32 == 8
    (257, 2064, 5, 16),      # chunk groups, n % 32 == 16
    (333, 2040, 3, 40),      # chunk groups straddling lanes, n % 32 == 24
    (700, 4104, 4, 72),      # chunk groups, several slices
    (900, 4104, 3, 4104),    # row-wise, n % 32 != 0
    (61, 8, 1, 8),           # the smallest n
]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def pack(d):
    import paper_2206_09557_b200 as L
    return L.lutgemm_pack_bcq(dev(d["planes"].view(np.int32)), dev(d["alpha"]),
                              None if d["offset"] is None else dev(d["offset"]), d["n"], d["g"])


def run(w, X):
    import paper_2206_09557_b200 as L
    Xd = dev(np.atleast_2d(X))
    y = L.lutgemm_gemv(w, Xd[0])[None] if Xd.shape[0] == 1 else L.lutgemm_gemm_batched(w, Xd)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("off", [False, True])
@pytest.mark.parametrize("m,n,q,g", SHAPES)
def test_general_shape_gemv_and_batched(m, n, q, g, off):
    d = gen_bcq(m + 7 * n + q, m, n, q, g, offset=off)
    w = pack(d)
    for b in (1, 2, 3, 6):
        X = gen_x(b * 31 + n, b, n)
        ref = O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g)
        assert_parity(run(w, X), ref, (m, n, q, g, off, b))


@pytest.mark.parametrize("m,n,q,g", SHAPES[:4] + SHAPES[4:6])
def test_general_shape_round_trip(m, n, q, g):
    import paper_2206_09557_b200 as L
    d = gen_bcq(m + n, m, n, q, g, offset=True)
    p, a, z = L.lutgemm_unpack_bcq(pack(d))
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy().view(np.uint32), d["planes"])
    assert np.array_equal(a.cpu().numpy().view(np.uint16), d["alpha"].view(np.uint16))
    assert np.array_equal(z.cpu().numpy().view(np.uint16), d["offset"].view(np.uint16))


@pytest.mark.parametrize("m,n,q,g,compact", [(600, 4104, 4, 24, False), (600, 4800, 4, 96, True),
                                             (600, 4800, 4, 96, False), (300, 2040, 3, 40, False)])
def test_general_shape_uniform(m, n, q, g, compact):
    """App. C conversion for the general group sizes; the compact format takes the
    straddling class (g % 32 == 0), the chunk class is packed in the expanded format."""
    import paper_2206_09557_b200 as L
    u = gen_uniform(m + n + q, m, n, q, g)
    w = L.lutgemm_pack_uniform(dev(u["codes"]), dev(u["scale"]), dev(u["zero"]), q, g, compact=compact)
    planes, alpha, z = O.uniform_to_bcq(u["codes"], u["scale"], u["zero"], q)
    for b in (1, 4, 8):
        X = gen_x(b + m, b, n)
        ref = O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(z), X, n, g)
        assert_parity(run(w, X), ref, (m, n, q, g, compact, b))


@pytest.mark.parametrize("m,n,q,g", [(1000, 4800, 3, 96), (1029, 4104, 3, 24)])
def test_general_shape_p2p_world1(m, n, q, g):
    """The fused TP epilogue runs the same GEMV kernel: rows all-gather and column all-reduce at
    world 1 for a straddling and a chunk-group shape (m padded to the epilogue's 8-row units)."""
    import paper_2206_09557_b200 as L
    m8 = (m + 7) // 8 * 8
    d = gen_bcq(m + q, m8, n, q, g)
    w = pack(d)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(m8, n, 1), "cuda")
    grp = L.P2PGroup(0, 1, rows_out=m8, cols_m=m8)
    X = gen_x(m, 1, n)
    ref = O.bcq_gemv(d["planes"], d["alpha"], None, X, n, g)
    for fn in (grp.gemv_allgather, grp.gemv_allreduce):
        y = torch.empty(m8, dtype=torch.float16, device="cuda")
        fn(w, dev(X[0]), ws, y)
        torch.cuda.synchronize()
        assert_parity(y.float().cpu().numpy()[None], ref, (m, n, q, g, fn.__name__))
    grp.close()
