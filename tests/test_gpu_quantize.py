"""GPU quantizers vs the plain fp64 quantizer oracle
(oracle/quantize_plain.py) under the tie rule of DESIGN.md RQ5: codes, scales,
bit-planes and alphas bit-equal on every (row, group) whose decisions all clear the
float32 error bound, fragile groups counted and capped, their reconstruction error
bounded; the end-to-end chain dense W -> quantize -> pack -> LUT-GEMV against the
oracle product of the plain oracle's quantization.  Diagnostic: bit-exactness
against the mirrored-order replay (oracle/quantize_oracle.py)."""
import numpy as np
import pytest
import torch

import oracle as O
import oracle.quantize_oracle as Q
import oracle.quantize_plain as P
from tests._helpers import assert_parity, check_bcq_rule, check_rtn_rule
from workloads import gen_x

pytestmark = pytest.mark.gpu


def dense(seed, m, n, scale=0.05):
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((m, n)) * scale
    W[:, :32] += 0.3 * rng.standard_normal((m, 1))  # some offset groups
    W[0, :32] = 0.25  # a constant group (RTN degenerate case)
    return W.astype(np.float16)


SHAPES_RTN = [(7, 64, 1, 32), (33, 256, 2, 64), (16, 512, 3, 128), (9, 1024, 4, 1024), (5, 2048, 8, 256),
              (3, 3072, 4, 3072), (128, 1024, 3, 128)]
SHAPES_BCQ = [(7, 64, 1, 32), (33, 256, 2, 64), (16, 512, 3, 128), (9, 1024, 4, 1024), (4, 512, 6, 64),
              (3, 3072, 3, 3072), (96, 1024, 3, 128)]


@pytest.mark.parametrize("m,n,q,g", SHAPES_RTN)
def test_rtn_vs_plain_oracle(m, n, q, g):
    import paper_2206_09557_b200 as L
    W = dense(m + n, m, n)
    got = [t.cpu().numpy() for t in L.lutgemm_quantize_rtn(torch.from_numpy(W).cuda(), q, g)]
    rc, rs, rz, fragile = P.quantize_rtn(W, q, g)
    share = check_rtn_rule(got, (rc, rs, rz), fragile, W, q, g, cap=max(0.05, 3.0 / fragile.size))
    print(f"RTN {m}x{n} q={q} g={g}: fragile share {share:.4f}")


@pytest.mark.parametrize("iters", [0, 1, 3])
@pytest.mark.parametrize("m,n,q,g", SHAPES_BCQ)
def test_bcq_vs_plain_oracle(m, n, q, g, iters):
    import paper_2206_09557_b200 as L
    W = dense(m * q + n, m, n)
    gp, ga = (t.cpu().numpy() for t in L.lutgemm_quantize_bcq(torch.from_numpy(W).cuda(), q, g, iters))
    if iters == 0:
        rp, ra, fragile = P.quantize_bcq_greedy(W, q, g)
    else:
        rp, ra, fragile = P.quantize_bcq_alternating(W, q, g, iters)
    share = check_bcq_rule((gp.view(np.uint32), ga), (rp, ra), fragile, W, q, g,
                           cap=max(0.05, 3.0 / fragile.size))
    print(f"BCQ {m}x{n} q={q} g={g} iters={iters}: fragile share {share:.4f}")


@pytest.mark.parametrize("m,n,q,g", [(7, 64, 1, 32), (33, 256, 2, 64), (16, 512, 3, 128), (9, 1024, 4, 1024),
                                     (5, 2048, 8, 256), (3, 3072, 4, 3072)])
def test_rtn_bit_exact(m, n, q, g):
    """Diagnostic: bit-exact against the mirrored-order replay."""
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
    """Diagnostic: bit-exact against the mirrored-order replay."""
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
    plain oracle's quantization of the same W (fragile groups may differ by a level: within tolerance)."""
    import paper_2206_09557_b200 as L
    m, n, q, g = 1000, 2048, 3, 128
    W = dense(17, m, n)
    Wd = torch.from_numpy(W).cuda()
    X = gen_x(23, 4, n)
    if method.startswith("rtn"):
        c, s, z = L.lutgemm_quantize_rtn(Wd, q, g)
        w = L.lutgemm_pack_uniform(c, s, z, q, g, compact=method == "rtn_compact")
        rc, rs, rz, _ = P.quantize_rtn(W, q, g)
        planes, alpha, zz = O.uniform_to_bcq(rc, rs, rz, q)
        ref = O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(zz), X, n, g)
    else:
        iters = 0 if method == "greedy" else 2
        p, a = L.lutgemm_quantize_bcq(Wd, q, g, iters)
        w = L.lutgemm_pack_bcq(p, a, None, n, g)
        rp, ra, _ = P.quantize_bcq_greedy(W, q, g) if iters == 0 else P.quantize_bcq_alternating(W, q, g, iters)
        ref = O.bcq_gemv(rp, ra, None, X, n, g)
    Xd = torch.from_numpy(X).cuda()
    y1 = L.lutgemm_gemv(w, Xd[0]).float().cpu().numpy().astype(np.float64)
    yb = L.lutgemm_gemm_batched(w, Xd).float().cpu().numpy().astype(np.float64)
    assert_parity(y1[None], ref[:1], (method, 1))
    assert_parity(yb, ref, (method, 4))
