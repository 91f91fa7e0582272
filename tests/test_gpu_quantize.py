"""GPU quantizers vs the quantizer oracle: codes, scales, bit-planes
and alphas bit-exact (both sides take every integer decision in the same fp32 /
fp64 operation order), and the end-to-end chain dense W -> quantize
-> pack -> LUT-GEMV against the oracle product of the oracle's quantization."""
import numpy as np
import pytest
import torch

import oracle as O
import oracle.quantize_oracle as Q
from tests._helpers import assert_parity
from workloads import gen_x

pytestmark = pytest.mark.gpu


def dense(seed, m, n, scale=0.05):
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((m, n)) * scale
    W[:, :32] += 0.3 * rng.standard_normal((m, 1))  # some offset groups
    W[0, :32] = 0.25  # a constant group (RTN degenerate case)
    return W.astype(np.float16)


@pytest.mark.parametrize("m,n,q,g", [(7, 64, 1, 32), (33, 256, 2, 64), (16, 512, 3, 128), (9, 1024, 4, 1024),
                                     (5, 2048, 8, 256), (3, 3072, 4, 3072)])
def test_rtn_bit_exact(m, n, q, g):
    import paper_2206_09557_b200 as L
    W = dense(m + n, m, n)
    c, s, z = L.lutgemm_quantize_rtn(torch.from_numpy(W).cuda(), q, g)
    rc, rs, rz = Q.quantize_rtn(W, q, g)
    assert np.array_equal(c.cpu().numpy(), rc)
    assert np.array_equal(s.cpu().numpy().view(np.uint16), rs.view(np.uint16))
    assert np.array_equal(z.cpu().numpy().view(np.uint16), rz.view(np.uint16))


@pytest.mark.parametrize("iters", [0, 1, 3])
@pytest.mark.parametrize("m,n,q,g", [(7, 64, 1, 32), (33, 256, 2, 64), (16, 512, 3, 128), (9, 1024, 4, 1024),
                                     (4, 512, 6, 64), (3, 3072, 3, 3072)])
def test_bcq_bit_exact(m, n, q, g, iters):
    import paper_2206_09557_b200 as L
    W = dense(m * q + n, m, n)
    p, a = L.lutgemm_quantize_bcq(torch.from_numpy(W).cuda(), q, g, iters)
    if iters == 0:
        rp, ra = Q.quantize_bcq_greedy(W, q, g)
    else:
        rp, ra = Q.quantize_bcq_alternating(W, q, g, iters)
    assert np.array_equal(p.cpu().numpy().view(np.uint32), rp)
    assert np.array_equal(a.cpu().numpy().view(np.uint16), ra.view(np.uint16))


@pytest.mark.parametrize("method", ["rtn", "rtn_compact", "greedy", "alternating"])
def test_quantize_pack_gemv_chain(method):
    """dense W -> GPU quantizer -> lutgemm_pack_bcq -> GEMV (b = 1 and 4) == oracle product of the
    oracle's quantization of the same W."""
    import paper_2206_09557_b200 as L
    m, n, q, g = 1000, 2048, 3, 128
    W = dense(17, m, n)
    Wd = torch.from_numpy(W).cuda()
    X = gen_x(23, 4, n)
    if method.startswith("rtn"):
        c, s, z = L.lutgemm_quantize_rtn(Wd, q, g)
        w = L.lutgemm_pack_uniform(c, s, z, q, g, compact=method == "rtn_compact")
        rc, rs, rz = Q.quantize_rtn(W, q, g)
        planes, alpha, zz = O.uniform_to_bcq(rc, rs, rz, q)
        ref = O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(zz), X, n, g)
    else:
        iters = 0 if method == "greedy" else 2
        p, a = L.lutgemm_quantize_bcq(Wd, q, g, iters)
        w = L.lutgemm_pack_bcq(p, a, None, n, g)
        rp, ra = Q.quantize_bcq_greedy(W, q, g) if iters == 0 else Q.quantize_bcq_alternating(W, q, g, iters)
        ref = O.bcq_gemv(rp, ra, None, X, n, g)
    Xd = torch.from_numpy(X).cuda()
    y1 = L.lutgemm_gemv(w, Xd[0]).float().cpu().numpy().astype(np.float64)
    yb = L.lutgemm_gemm_batched(w, Xd).float().cpu().numpy().astype(np.float64)
    assert_parity(y1[None], ref[:1], (method, 1))
    assert_parity(yb, ref, (method, 4))
