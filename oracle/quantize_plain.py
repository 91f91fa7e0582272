"""Plain fp64 quantizer oracle -- TEST INFRASTRUCTURE ONLY.

Same import rules as ``bcq_oracle.py`` (tests/, smoke() and bench.py only); shares
no code with the CUDA quantizer kernels and none with ``quantize_oracle.py`` (the
mirrored-order replay, kept as a diagnostic).  This module is the DEFINITION the
GPU quantizers are checked against: every quantity in float64, every sum a plain
numpy sum, the least-squares step ``numpy.linalg.lstsq``, the nearest-level step
an argmin over all 2^q levels.

* ``quantize_rtn``: min-max RTN per (row, group) (the RTN baseline of Tables 3/6;
  SPEC S:L112-120): s = (max - min)/(2^q - 1) and z_hat = min, both stored fp16
  (round to nearest even), code = clamp(round_half_even((w - z_hat16)/s16)) from
  the stored values (RQ1, RQ2); a constant group stores s = 1, code 0.
* ``quantize_bcq_greedy``: w ~ sum_i alpha_i b_i (Sec. 2.3) fitted
  greedily on the residual: b_i = sign(r) with sign(0) = +1, alpha_i =
  fp16(mean |r|), r <- r - alpha_i b_i with the stored alpha (RQ3).
* ``quantize_bcq_alternating``: App. E's "iterative solver", RQ4: greedy
  start, then per round (a) alpha = lstsq(B^T, w) stored fp16 -- if B B^T is
  rank-deficient (two planes equal or opposite) the previous alpha is kept --
  and (b) every element's signs = the pattern whose level sum_i +-alpha_i is
  nearest to w (lowest pattern index on exact ties).

Tie rule (RQ5).  The GPU takes the same decisions in float32 (sums in a
lane/butterfly order) where this oracle uses float64, so a decision whose float64
margin is below the float32 rounding error the kernel can make may legitimately
go the other way.  Every decision here also returns its margin against a bound on
that error (u = 2^-24; a float32 sum's error is bounded by 6 sigma of the
probabilistic rounding model over the partial sums the kernel forms, ``_sum_err``;
single operations by their worst case):

* fp16 storage of a value v (alpha, s): the distance from v to the nearest fp16
  rounding midpoint is compared with the value's error bound;
* a sign b = sign(r): |r| against the residual's error bound;
* a nearest level: the gap between the best and second-best |w - v_k|;
* a rounded code: the distance of (w - z)/s to the nearest half-integer;
* a least-squares step: the fp16 rounding margins of alpha against
  |G^-1| (d u sum|w|) (G = B B^T), and pivots of G below 1 (the kernel's
  singularity threshold is pivot <= 0.5).

A (row, group) with any decision inside its bound is FRAGILE: its outputs may
differ from the GPU's (and everything downstream in that group with them).  The
tests require bit equality on every non-fragile group, cap the fragile share, and
bound the reconstruction error of the fragile groups.
"""
from __future__ import annotations

import numpy as np

__all__ = ["quantize_rtn", "quantize_bcq_greedy", "quantize_bcq_alternating", "fp16_round_margin"]

U32 = 2.0 ** -24  # float32 unit roundoff


def _groups(n: int, g: int):
    return [(c0, min(n, c0 + g)) for c0 in range(0, n, g)]


def _sum_err(x: np.ndarray) -> float:
    """Error bound of the kernel's float32 sum of x: lane l adds x[l], x[l+32], ... in order, then
    5 butterfly levels combine the 32 lane sums.  Each addition rounds its partial sum p with
    relative error <= u; treating the roundings as independent and uniform (probabilistic
    error analysis) the total error has sigma = u sqrt(sum p^2 / 3), and the bound is 6 sigma
    (a 6-sigma event for the GPU's float32 error to exceed it).  If x holds float32 values and
    every partial sum is itself a float32 value, the kernel's sum is exact: the bound is 0."""
    x = np.asarray(x, dtype=np.float64)
    L = x.shape[0]
    pad = np.zeros(-(-L // 32) * 32)
    pad[:L] = x
    lanes = np.cumsum(pad.reshape(-1, 32), axis=0)          # partial sums of every lane
    sq = float(np.sum(lanes[1:] ** 2))                       # the first term of a lane is not rounded
    exact = _is_f32(pad) and _is_f32(lanes)
    v = lanes[-1]
    for o in (16, 8, 4, 2, 1):                               # butterfly: v[l] + v[l ^ o]
        v = v + v[np.arange(32) ^ o]
        sq += float(np.sum(v ** 2)) / 32                     # lane 0's chain (one sum per level)
        exact = exact and _is_f32(v)
    return 0.0 if exact else 6 * U32 * np.sqrt(sq / 3)


def _is_f32(a) -> bool:
    a = np.asarray(a, dtype=np.float64)
    return bool(np.all(a.astype(np.float32).astype(np.float64) == a))


def fp16_round_margin(v: float) -> float:
    """Absolute distance from v to the nearest fp16 rounding boundary (the midpoint between
    the two fp16 values around v): how far v may move before fp16(v) changes."""
    v = float(v)
    h = np.float16(v)
    hv = float(h)
    if not np.isfinite(hv):
        return 0.0
    up = float(np.nextafter(h, np.float16(np.inf)))
    dn = float(np.nextafter(h, np.float16(-np.inf)))
    # fp16(v) = h: v lies in [mid(dn, h), mid(h, up)]
    return min(abs(v - 0.5 * (hv + up)), abs(v - 0.5 * (hv + dn)))


def _pack(planes, r, c0, signs_i, i):
    for j, s in enumerate(signs_i):
        if s:
            c = c0 + j
            planes[i, r, c // 32] |= np.uint32(1) << np.uint32(c % 32)


# ---------------------------------------------------------------------------
# RTN
# ---------------------------------------------------------------------------

def rtn_group(w: np.ndarray, q: int):
    """One group: returns (codes int [len], s16, z16, fragile)."""
    w = np.asarray(w, dtype=np.float64)
    mn, mx = float(w.min()), float(w.max())
    z16 = np.float16(mn)  # exact: w holds fp16 values
    if mx == mn:
        return np.zeros(w.shape[0], dtype=np.int64), np.float16(1.0), z16, False
    s = (mx - mn) / (2 ** q - 1)
    # kernel: d = mx - mn and s = d / (2^q - 1) in float32; each is exact when its exact value is a
    # float32 value, else within u (relative) of it
    d = mx - mn
    err_s = (0.0 if _is_f32(d) else U32 * s) + (0.0 if (_is_f32(d) and _is_f32(s)) else U32 * s)
    fragile = fp16_round_margin(s) < err_s if err_s > 0 else False
    s16 = np.float16(s)
    t = (w - float(z16)) / float(s16)
    codes = np.clip(np.rint(t), 0, 2 ** q - 1).astype(np.int64)
    # kernel: (w - z_hat) (exact: fp16 operands) / s in float32 -> exact when t is a float32 value,
    # else within u |t|; an exact half-integer is rounded half-to-even on both sides
    t32_exact = t.astype(np.float32).astype(np.float64) == t
    err_t = np.where(t32_exact, 0.0, 2 * U32 * (np.abs(t) + 1.0))
    half_gap = np.abs(t - (np.floor(t) + 0.5))
    inside = (t > -0.5) & (t < 2 ** q - 0.5)
    fragile |= bool(np.any(inside & (half_gap <= err_t) & (err_t > 0)))
    return codes, s16, z16, bool(fragile)


def quantize_rtn(W: np.ndarray, q: int, g: int):
    """Returns codes uint8 [m][n], scale fp16 [m][G], zero fp16 [m][G], fragile bool [m][G]."""
    W = np.asarray(W, dtype=np.float16)
    m, n = W.shape
    grp = _groups(n, g)
    codes = np.zeros((m, n), dtype=np.uint8)
    scale = np.zeros((m, len(grp)), dtype=np.float16)
    zero = np.zeros((m, len(grp)), dtype=np.float16)
    fragile = np.zeros((m, len(grp)), dtype=bool)
    for r in range(m):
        for k, (c0, c1) in enumerate(grp):
            c, s16, z16, fr = rtn_group(W[r, c0:c1], q)
            codes[r, c0:c1] = c
            scale[r, k], zero[r, k], fragile[r, k] = s16, z16, fr
    return codes, scale, zero, fragile


# ---------------------------------------------------------------------------
# greedy BCQ
# ---------------------------------------------------------------------------

def greedy_group(w: np.ndarray, q: int):
    """One group: returns (alpha fp16 [q], signs bool [q][len], fragile, residual-error bound [len])."""
    w = np.asarray(w, dtype=np.float64)
    L = w.shape[0]
    r = w.copy()
    err_r = np.zeros(L)             # bound on the kernel's float32 residual error
    alpha = np.zeros(q, dtype=np.float16)
    signs = np.zeros((q, L), dtype=bool)
    fragile = False
    for i in range(q):
        b = r >= 0
        fragile |= bool(np.any((err_r > 0) & (np.abs(r) <= err_r)))
        a = float(np.sum(np.abs(r))) / L
        # the kernel: float32 sum of |r|, divided by L (exact for a power-of-two L of exact operands)
        err_a = (_sum_err(np.abs(r)) + 6 * float(np.sqrt(np.sum(err_r ** 2) / 3))) / L
        if err_a > 0 or not _is_f32(a):
            err_a += U32 * a
        fragile |= fp16_round_margin(a) <= err_a
        a16 = np.float16(a)
        r = np.where(b, r - float(a16), r + float(a16))
        # float32 update r -= +-alpha: exact when the operands are and the result is a float32 value
        inexact = (err_r > 0) | (r.astype(np.float32).astype(np.float64) != r)
        err_r = np.where(inexact, err_r + U32 * (np.abs(r) + float(a16)), 0.0)
        alpha[i], signs[i] = a16, b
    return alpha, signs, bool(fragile)


def quantize_bcq_greedy(W: np.ndarray, q: int, g: int):
    """Returns planes uint32 [q][m][ceil(n/32)], alpha fp16 [m][G][q], fragile bool [m][G]."""
    W = np.asarray(W, dtype=np.float16)
    m, n = W.shape
    grp = _groups(n, g)
    planes = np.zeros((q, m, (n + 31) // 32), dtype=np.uint32)
    alpha = np.zeros((m, len(grp), q), dtype=np.float16)
    fragile = np.zeros((m, len(grp)), dtype=bool)
    for r in range(m):
        for k, (c0, c1) in enumerate(grp):
            a, s, fr = greedy_group(W[r, c0:c1], q)
            alpha[r, k], fragile[r, k] = a, fr
            for i in range(q):
                _pack(planes, r, c0, s[i], i)
    return planes, alpha, fragile


# ---------------------------------------------------------------------------
# alternating BCQ
# ---------------------------------------------------------------------------

def lstsq_alpha(signs: np.ndarray, w: np.ndarray, prev16: np.ndarray):
    """(a) alpha = argmin ||w - B^T alpha||_2 (numpy.linalg.lstsq), B = +-1 [q][len]; rank-deficient
    B B^T keeps the previous alpha.  Returns (alpha16, fragile)."""
    q, L = signs.shape
    B = np.where(signs, 1.0, -1.0)
    G = B @ B.T
    if np.linalg.matrix_rank(G) < q:
        return prev16.copy(), False
    # leading minors are integers; a pivot D_k / D_{k-1} below 1 is near the kernel's 0.5 threshold
    D = [1.0] + [round(float(np.linalg.det(G[:k, :k]))) for k in range(1, q + 1)]
    fragile = any(0 < D[k] / D[k - 1] < 1.0 for k in range(1, q + 1))
    alpha = np.linalg.lstsq(B.T, w, rcond=None)[0]
    err_c = max(_sum_err(B[i] * w) for i in range(q))
    err_alpha = np.abs(np.linalg.inv(G)).sum(axis=1) * err_c + 1e-12 * np.abs(alpha)
    fragile |= any(fp16_round_margin(alpha[i]) <= err_alpha[i] for i in range(q))
    return alpha.astype(np.float16), bool(fragile)


def nearest_signs(w: np.ndarray, alpha16: np.ndarray):
    """(b) per element the pattern k (bit i = sign of plane i) minimising |w - sum_i +-alpha_i|,
    the lowest k on exact ties.  Returns (signs bool [q][len], fragile)."""
    q = alpha16.shape[0]
    a = alpha16.astype(np.float64)
    K = 2 ** q
    bits = (np.arange(K)[:, None] >> np.arange(q)[None, :]) & 1           # [K][q]
    levels = np.where(bits == 1, 1.0, -1.0) @ a                           # [K]
    err = np.abs(w[:, None] - levels[None, :])                            # [len][K]
    best = np.argmin(err, axis=1)
    srt = np.sort(err, axis=1)
    gap = srt[:, 1] - srt[:, 0]
    # kernel: levels summed in float32 in plane order and |w - v| in float32; when every level
    # and every |w - v| is a float32 value those are exact and the comparison is too (exact
    # ties go to the lowest k on both sides)
    exact = _is_f32(np.cumsum(np.where(bits == 1, 1.0, -1.0) * a[None, :], axis=1)) and _is_f32(err)
    bound = 0.0 if exact else 2 * (q + 2) * U32 * (np.abs(w) + np.sum(np.abs(a)))
    fragile = bool(np.any((gap <= bound) & (bound > 0)))
    return np.array([(best >> i) & 1 for i in range(q)], dtype=bool), fragile


def quantize_bcq_alternating(W: np.ndarray, q: int, g: int, iters: int):
    """Greedy start, then `iters` rounds of (a) lstsq alpha and (b) nearest sign patterns.
    Returns planes, alpha fp16 [m][G][q], fragile bool [m][G]."""
    W = np.asarray(W, dtype=np.float16)
    m, n = W.shape
    grp = _groups(n, g)
    planes = np.zeros((q, m, (n + 31) // 32), dtype=np.uint32)
    alpha = np.zeros((m, len(grp), q), dtype=np.float16)
    fragile = np.zeros((m, len(grp)), dtype=bool)
    for r in range(m):
        for k, (c0, c1) in enumerate(grp):
            w = W[r, c0:c1].astype(np.float64)
            a16, s, fr = greedy_group(w, q)
            for _ in range(iters):
                a16, f1 = lstsq_alpha(s, w, a16)
                s, f2 = nearest_signs(w, a16)
                fr |= f1 or f2
            alpha[r, k], fragile[r, k] = a16, fr
            for i in range(q):
                _pack(planes, r, c0, s[i], i)
    return planes, alpha, fragile
