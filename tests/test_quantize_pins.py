"""Pins of the quantizer oracle (oracle/quantize_oracle.py) against
SPEC examples, closed forms, an independent least-squares routine
and brute force -- CPU only."""
import itertools

import numpy as np
import pytest

import oracle.quantize_oracle as Q
from oracle import dequantize, unpack_signs


def deq(planes, alpha, n, g):
    return dequantize(planes, alpha, None, n, g)


# ---- RTN ----

def test_rtn_spec_examples():
    c, s, z = Q.quantize_rtn(np.array([[0.0, 1.0]]), 1, 2)
    assert c.tolist() == [[0, 1]] and float(s[0, 0]) == 1.0 and float(z[0, 0]) == 0.0
    c, s, z = Q.quantize_rtn(np.array([[-1.0, 0.0, 1.0]]), 2, 3)
    assert float(s[0, 0]) == float(np.float16(2 / 3)) and float(z[0, 0]) == -1.0 and c.tolist() == [[0, 2, 3]]
    c, s, z = Q.quantize_rtn(np.array([[5.0, 5.0]]), 3, 2)  # degenerate group
    assert c.tolist() == [[0, 0]] and float(s[0, 0]) == 1.0 and float(z[0, 0]) == 5.0
    W = s[0, 0].astype(np.float64) * c + z[0, 0].astype(np.float64)
    assert np.array_equal(W, [[5.0, 5.0]])


@pytest.mark.parametrize("q,g", [(2, 32), (3, 64), (4, 128)])
def test_rtn_codes_are_nearest_levels(q, g):
    """Every code is the nearest of the 2^q levels s*c + z (brute force over all c)."""
    rng = np.random.default_rng(q * g)
    W = rng.standard_normal((6, 4 * g)).astype(np.float16)
    codes, s, z = Q.quantize_rtn(W, q, g)
    for r in range(W.shape[0]):
        for k in range(W.shape[1] // g):
            w = W[r, k * g:(k + 1) * g].astype(np.float64)
            lv = s[r, k].astype(np.float64) * np.arange(2 ** q) + z[r, k].astype(np.float64)
            err = np.abs(w[:, None] - lv[None, :])
            got = err[np.arange(g), codes[r, k * g:(k + 1) * g]]
            assert np.all(got <= err.min(axis=1) + 1e-3 * float(s[r, k]))  # ties / fp32 rounding only
            # min maps to code 0 and max to the top code (up to fp16 rounding of s and z)
            assert codes[r, k * g + int(np.argmin(w))] == 0


# ---- greedy BCQ ----

def test_greedy_spec_examples():
    p, a = Q.quantize_bcq_greedy(np.array([[1.0, -1.0]]), 1, 2)
    assert float(a[0, 0, 0]) == 1.0 and unpack_signs(p, 2)[0, 0].tolist() == [1, -1]
    p, a = Q.quantize_bcq_greedy(np.array([[3.0, 1.0]]), 2, 2)
    assert a[0, 0].tolist() == [2.0, 1.0]
    sg = unpack_signs(p, 2)
    assert sg[0, 0].tolist() == [1, 1] and sg[1, 0].tolist() == [1, -1]
    assert np.array_equal(deq(p, a, 2, 2), [[3.0, 1.0]])  # exact reconstruction


def test_greedy_one_bit_closed_form_and_monotone_residual():
    rng = np.random.default_rng(5)
    W = rng.standard_normal((8, 128)).astype(np.float16)
    p, a = Q.quantize_bcq_greedy(W, 1, 32)
    for r in range(8):
        for k in range(4):
            w = W[r, 32 * k:32 * (k + 1)].astype(np.float64)
            assert abs(float(a[r, k, 0]) - np.mean(np.abs(w))) <= 1e-3 * np.mean(np.abs(w))  # fp16 of mean|w|
    prev = None
    for q in (1, 2, 3, 4):
        p, a = Q.quantize_bcq_greedy(W, q, 32)
        e = Q.quantization_error(W, deq(p, a, 128, 32))["mse"]
        assert prev is None or e < prev
        prev = e


def test_greedy_scale_equivariance():
    rng = np.random.default_rng(6)
    W = (rng.standard_normal((4, 64)) * 0.5).astype(np.float16)
    p1, a1 = Q.quantize_bcq_greedy(W, 3, 32)
    p2, a2 = Q.quantize_bcq_greedy((2 * W.astype(np.float32)).astype(np.float16), 3, 32)
    assert np.array_equal(p1, p2) and np.array_equal(2 * a1.astype(np.float32), a2.astype(np.float32))


# ---- alternating BCQ (App. E) ----

def test_alternating_spec_examples():
    w = np.array([[0.9, 1.1, -1.0]])
    p, a = Q.quantize_bcq_alternating(w, 1, 3, 2)
    assert float(a[0, 0, 0]) == float(np.float16(1.0)) and unpack_signs(p, 3)[0, 0].tolist() == [1, 1, -1]
    rng = np.random.default_rng(7)
    W = rng.standard_normal((4, 64)).astype(np.float16)
    assert all(np.array_equal(x, y) for x, y in zip(Q.quantize_bcq_alternating(W, 1, 32, 3),
                                                    Q.quantize_bcq_greedy(W, 1, 32)))


def test_alternating_least_squares_step_matches_lstsq():
    rng = np.random.default_rng(8)
    for q in (2, 3, 4):
        signs = rng.random((q, 64)) < 0.5
        w = rng.standard_normal(64).astype(np.float32)
        x = Q._solve_alpha(signs, w, np.zeros(q))
        B = np.where(signs, 1.0, -1.0).T
        ref = np.linalg.lstsq(B, w.astype(np.float64), rcond=None)[0]
        assert np.allclose(x, ref, rtol=1e-5, atol=1e-7)


def test_alternating_nearest_step_brute_force():
    rng = np.random.default_rng(9)
    for q in (1, 2, 3):
        a16 = np.sort(rng.random(q).astype(np.float16))[::-1].copy()
        w = rng.standard_normal(40).astype(np.float32)
        s = Q._nearest_signs(w, a16)
        for t in range(40):
            best = min(abs(float(w[t]) - sum(float(a16[i]) * (1 if bb[i] else -1) for i in range(q)))
                       for bb in itertools.product([False, True], repeat=q))
            got = abs(float(w[t]) - sum(float(a16[i]) * (1 if s[i, t] else -1) for i in range(q)))
            assert got <= best + 1e-6


@pytest.mark.parametrize("q", [2, 3, 4])
def test_alternating_not_worse_than_greedy(q):
    rng = np.random.default_rng(10 + q)
    W = rng.standard_normal((16, 64)).astype(np.float16)
    pg, ag = Q.quantize_bcq_greedy(W, q, 32)
    pa, aa = Q.quantize_bcq_alternating(W, q, 32, 3)
    for r in range(16):
        for k in range(2):
            sl = slice(32 * k, 32 * (k + 1))
            eg = Q.quantization_error(W[r:r + 1, sl], deq(pg[:, r:r + 1, k:k + 1], ag[r:r + 1, k:k + 1], 32, 32))["mse"]
            ea = Q.quantization_error(W[r:r + 1, sl], deq(pa[:, r:r + 1, k:k + 1], aa[r:r + 1, k:k + 1], 32, 32))["mse"]
            assert ea <= eg * (1 + 2e-3) + 1e-12  # fp16 storage of alpha may cost a hair


def test_alternating_recovers_an_exact_bcq_matrix():
    """w = sum_i alpha_i b_i exactly (fp16 alphas, random signs): alternating
    reaches zero error (LS returns the true alphas, the nearest step the true signs)."""
    rng = np.random.default_rng(11)
    al = np.array([0.5, 0.25, 0.125])
    signs = rng.random((3, 8, 64)) < 0.5
    W = np.einsum("i,irc->rc", al, np.where(signs, 1.0, -1.0)).astype(np.float16)
    p, a = Q.quantize_bcq_alternating(W, 3, 64, 4)
    assert Q.quantization_error(W, deq(p, a, 64, 64))["max_abs"] == 0.0


# ---- error metric and order of the fixed-order sum ----

def test_quantization_error_and_lane_sum():
    e = Q.quantization_error(np.array([[1.0]]), np.array([[0.5]]))
    assert e == {"mse": 0.25, "rel_fro": 0.5, "max_abs": 0.5}
    assert Q.quantization_error(np.ones((2, 2)), np.ones((2, 2)))["mse"] == 0.0
    v = np.arange(1, 101, dtype=np.float32)
    assert float(Q.lane_sum_f32(v)) == 5050.0  # exact for small integers in any order
