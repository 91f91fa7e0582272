"""GPU pack path: native bytes equal an independent numpy packer, the
native -> canonical round trip is bit-exact, and the uniform -> BCQ pack
(App. C) stores exactly the oracle's fp16-rounded alpha and z."""
import numpy as np
import pytest
import torch

import oracle as O
from tests._helpers import native_pack_reference
from workloads import gen_bcq, gen_uniform

pytestmark = pytest.mark.gpu

SHAPES = [  # (m, n, q, g, offset): row tails, partial last slice, several slices, q/g range
    (4, 32, 1, 32, False),
    (7, 96, 3, 32, True),
    (37, 1056, 2, 32, False),
    (100, 1536, 3, 128, True),
    (64, 3072, 4, 1024, False),
    (13, 2048, 8, 2048, True),
    # SURVEY 8(b) shapes beyond powers of two: groups straddling slices, chunk groups, n % 32 != 0
    (9, 4800, 3, 96, True),
    (6, 4608, 2, 384, False),
    (5, 4608, 3, 1536, True),
    (7, 4104, 3, 24, True),
    (10, 1000, 2, 8, False),
    (3, 4104, 4, 4104, True),
    (130, 2560, 5, 64, True),
    (9, 1056, 3, 1056, True),
    (20, 4096, 2, 2048, False),
]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def pack(d):
    import paper_2206_09557_b200 as L
    return L.lutgemm_pack_bcq(dev(d["planes"].view(np.int32)), dev(d["alpha"]),
                              None if d["offset"] is None else dev(d["offset"]), d["n"], d["g"])


@pytest.mark.parametrize("m,n,q,g,off", SHAPES)
def test_pack_bytes_match_independent_packer(m, n, q, g, off):
    d = gen_bcq(m * 7 + n, m, n, q, g, offset=off)
    w = pack(d)
    torch.cuda.synchronize()
    ref = native_pack_reference(d["planes"], d["alpha"], d["offset"], m, n, q, g)
    assert np.array_equal(w.data.cpu().numpy(), ref)


@pytest.mark.parametrize("m,n,q,g,off", SHAPES)
def test_unpack_round_trip_bit_exact(m, n, q, g, off):
    import paper_2206_09557_b200 as L
    d = gen_bcq(m + 3 * n, m, n, q, g, offset=off)
    w = pack(d)
    p, a, z = L.lutgemm_unpack_bcq(w)
    torch.cuda.synchronize()
    assert np.array_equal(p.cpu().numpy().view(np.uint32), d["planes"])
    assert np.array_equal(a.cpu().numpy().view(np.uint16), d["alpha"].view(np.uint16))
    if off:
        assert np.array_equal(z.cpu().numpy().view(np.uint16), d["offset"].view(np.uint16))


@pytest.mark.parametrize("m,n,q,g", [(8, 64, 1, 32), (33, 256, 2, 64), (64, 512, 3, 128), (100, 1536, 4, 128),
                                     (17, 1024, 8, 256), (11, 4104, 4, 24), (6, 4800, 3, 96)])
@pytest.mark.parametrize("compact", [False, True])
def test_uniform_pack_matches_oracle_conversion(m, n, q, g, compact):
    """GPU App. C conversion == oracle.uniform_to_bcq followed by the fp16
    storage step, bit for bit (planes, alpha, z).  The compact format stores s
    and unpacks to alpha_i = 2^(i-1) s: the same canonical bytes."""
    import paper_2206_09557_b200 as L
    if compact and g % 32:
        pytest.skip("the compact format needs g % 32 == 0 (test_abi_cpu checks the rejection)")
    u = gen_uniform(m * n + q, m, n, q, g)
    w = L.lutgemm_pack_uniform(dev(u["codes"]), dev(u["scale"]), dev(u["zero"]), q, g, compact=compact)
    if compact:  # one fp16 scale per (row, group) instead of q
        assert w.nbytes() < L.lutgemm_packed_bytes(m, n, q, g, True) or q == 1
        assert w.fmt == L.FMT_UNIFORM_COMPACT
    p, a, z = L.lutgemm_unpack_bcq(w)
    torch.cuda.synchronize()
    planes, alpha, zz = O.uniform_to_bcq(u["codes"], u["scale"], u["zero"], q)
    assert np.array_equal(p.cpu().numpy().view(np.uint32), planes)
    assert np.array_equal(a.cpu().numpy().view(np.uint16), O.store_fp16(alpha).view(np.uint16))
    assert np.array_equal(z.cpu().numpy().view(np.uint16), O.store_fp16(zz).view(np.uint16))
