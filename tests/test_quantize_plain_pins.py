"""Pins of the plain fp64 quantizer oracle (oracle/quantize_plain.py, the definition the GPU
quantizers are checked against, RQ5) -- CPU only: SPEC examples,
closed forms, numpy.linalg.lstsq, brute force over all sign patterns, and the tie rule
exercised against the mirrored-order replay (oracle/quantize_oracle.py, which takes every
decision in the kernel's float32 order): every non-fragile group is bit-equal."""
import itertools

import numpy as np
import pytest

import oracle.quantize_oracle as M
import oracle.quantize_plain as P
from oracle import dequantize, unpack_signs
from tests._helpers import check_bcq_rule, check_rtn_rule


def deq(planes, alpha, n, g):
    return dequantize(planes, alpha, None, n, g)


def test_plain_rtn_spec_examples():
    c, s, z, fr = P.quantize_rtn(np.array([[0.0, 1.0]]), 1, 2)
    assert c.tolist() == [[0, 1]] and float(s[0, 0]) == 1.0 and float(z[0, 0]) == 0.0 and not fr.any()
    c, s, z, _ = P.quantize_rtn(np.array([[-1.0, 0.0, 1.0]]), 2, 3)
    assert float(s[0, 0]) == float(np.float16(2 / 3)) and float(z[0, 0]) == -1.0 and c.tolist() == [[0, 2, 3]]
    c, s, z, _ = P.quantize_rtn(np.array([[5.0, 5.0]]), 3, 2)  # constant group
    assert c.tolist() == [[0, 0]] and float(s[0, 0]) == 1.0 and float(z[0, 0]) == 5.0


@pytest.mark.parametrize("q,g", [(2, 32), (4, 128)])
def test_plain_rtn_codes_are_nearest_stored_levels(q, g):
    rng = np.random.default_rng(q + g)
    W = rng.standard_normal((5, 3 * g)).astype(np.float16)
    codes, s, z, _ = P.quantize_rtn(W, q, g)
    for r in range(5):
        for k in range(3):
            w = W[r, k * g:(k + 1) * g].astype(np.float64)
            lv = float(s[r, k]) * np.arange(2 ** q) + float(z[r, k])
            err = np.abs(w[:, None] - lv[None, :])
            got = err[np.arange(g), codes[r, k * g:(k + 1) * g]]
            assert np.all(got <= err.min(axis=1) + 1e-12)


def test_plain_greedy_spec_examples_and_closed_form():
    p, a, _ = P.quantize_bcq_greedy(np.array([[1.0, -1.0]]), 1, 2)
    assert float(a[0, 0, 0]) == 1.0 and unpack_signs(p, 2)[0, 0].tolist() == [1, -1]
    p, a, _ = P.quantize_bcq_greedy(np.array([[3.0, 1.0]]), 2, 2)
    assert a[0, 0].tolist() == [2.0, 1.0] and np.array_equal(deq(p, a, 2, 2), [[3.0, 1.0]])
    rng = np.random.default_rng(3)
    W = rng.standard_normal((4, 64)).astype(np.float16)
    p, a, _ = P.quantize_bcq_greedy(W, 1, 32)  # q = 1: alpha = fp16(mean |w|), b = sign(w)
    for r in range(4):
        for k in range(2):
            w = W[r, 32 * k:32 * (k + 1)].astype(np.float64)
            assert a[r, k, 0] == np.float16(np.mean(np.abs(w)))
            assert np.array_equal(unpack_signs(p, 64)[0, r, 32 * k:32 * (k + 1)], np.where(w >= 0, 1, -1))


def test_plain_alternating_spec_example_and_exact_recovery():
    p, a, _ = P.quantize_bcq_alternating(np.array([[0.9, 1.1, -1.0]]), 1, 3, 2)
    assert float(a[0, 0, 0]) == float(np.float16(1.0)) and unpack_signs(p, 3)[0, 0].tolist() == [1, 1, -1]
    rng = np.random.default_rng(11)
    al = np.array([0.5, 0.25, 0.125])
    signs = rng.random((3, 8, 64)) < 0.5
    W = np.einsum("i,irc->rc", al, np.where(signs, 1.0, -1.0)).astype(np.float16)
    p, a, _ = P.quantize_bcq_alternating(W, 3, 64, 4)
    assert np.array_equal(deq(p, a, 64, 64), W.astype(np.float64))


def test_plain_steps_against_brute_force():
    rng = np.random.default_rng(12)
    for q in (1, 2, 3):
        a16 = np.sort(rng.random(q).astype(np.float16))[::-1].copy()
        w = rng.standard_normal(40)
        s, _ = P.nearest_signs(w, a16)
        for t in range(40):
            best = min(abs(w[t] - sum(float(a16[i]) * (1 if bb[i] else -1) for i in range(q)))
                       for bb in itertools.product([False, True], repeat=q))
            got = abs(w[t] - sum(float(a16[i]) * (1 if s[i, t] else -1) for i in range(q)))
            assert got == best
        signs = rng.random((q, 64)) < 0.5
        a, _ = P.lstsq_alpha(signs, w[:32].repeat(2), np.zeros(q, np.float16))
        B = np.where(signs, 1.0, -1.0)
        # normal equations hold up to the fp16 storage of alpha
        ref = np.linalg.solve(B @ B.T, B @ w[:32].repeat(2)) if np.linalg.matrix_rank(B @ B.T) == q else None
        if ref is not None:
            assert np.all(np.abs(a.astype(np.float64) - ref) <= np.abs(ref) * 2 ** -11 + 2 ** -24)


def test_fp16_round_margin():
    assert P.fp16_round_margin(1.0) == pytest.approx(2 ** -12)          # half-ulp below 1 is 2^-12
    assert P.fp16_round_margin(1.0 + 2 ** -11) == 0.0                    # exactly a midpoint
    assert P.fp16_round_margin(1.0 + 2 ** -12) == pytest.approx(2 ** -12)


def _dense(seed, m, n, scale=0.05):
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((m, n)) * scale
    W[:, :32] += 0.3 * rng.standard_normal((m, 1))
    W[0, :32] = 0.25
    return W.astype(np.float16)


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("m,n,q,g", [(33, 256, 2, 64), (16, 512, 3, 128), (9, 1024, 4, 1024), (4, 512, 6, 64),
                                     (3, 3072, 3, 3072)])
def test_tie_rule_against_the_mirrored_replay(seed, m, n, q, g):
    """The mirrored replay decides exactly as the kernels do (bit-exact on the GPU, tests/
    test_gpu_quantize.py); the plain oracle's tie rule must accept it: bit-equal outside the
    fragile groups, fragile share capped (RQ5)."""
    W = _dense(seed * 1000 + m * q + n, m, n)
    ref = P.quantize_rtn(W, q, g)
    check_rtn_rule(M.quantize_rtn(W, q, g), ref[:3], ref[3], W, q, g, cap=0.05)
    rp, ra, fr = P.quantize_bcq_greedy(W, q, g)
    check_bcq_rule(M.quantize_bcq_greedy(W, q, g), (rp, ra), fr, W, q, g, cap=0.35)
    rp, ra, fr = P.quantize_bcq_alternating(W, q, g, 2)
    check_bcq_rule(M.quantize_bcq_alternating(W, q, g, 2), (rp, ra), fr, W, q, g, cap=0.35)
