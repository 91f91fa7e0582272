"""Quantizer oracle -- TEST INFRASTRUCTURE ONLY.

Plain CPU definitions of the offline step before the LUT-GEMM path: turning a
dense fp16 weight into the formats the path consumes.  Same import rules as
``bcq_oracle.py`` (tests/, smoke() and bench.py only); shares no code with the
CUDA quantizer kernels.

* ``quantize_rtn``   -- uniform min-max round-to-nearest per (row, group) (the
  RTN baseline of Tables 3/6, "RTN"; SPEC S:L112-120 for the conventions).  Its
  output feeds the App. C conversion.
* ``quantize_bcq_greedy`` -- w ~ sum_i alpha_i b_i (Sec. 2.3) built
  greedily on the residual: b_i = sign(r) (sign(0) = +1), alpha_i = mean |r|,
  r <- r - alpha_i b_i (the paper defers the constructor to
  Xu et al.).
* ``quantize_bcq_alternating`` -- the "iterative solver introduced in
  [Xu et al. 2018]" of App. E: greedy start, then `iters` rounds of
  (a) alpha = argmin ||w - B alpha|| for fixed B (least squares) and
  (b) every b column = the sign pattern whose level sum_i alpha_i b_i is nearest
  to w (exhaustive over the 2^q patterns).

Where floating point decides an integer (a code, a sign, the nearest level),
the decision is taken in the precision the GPU kernels use, with the same
operation order, so codes and bit-planes can be compared bit for bit:

* elements are the fp16 weights as float32 (exact);
* a per-group sum runs over 32 "lanes": lane l adds elements l, l+32, l+64, ...
  in order in float32, then the 32 partials combine by the butterfly
  p[l] <- p[l] + p[l ^ o] for o = 16, 8, 4, 2, 1 (float32);
* RTN: s = fp16((max - min) / (2^q - 1)) and z_hat = fp16(min) are rounded to
  fp16 FIRST and codes are computed from the stored values,
  code = clamp(rint((w - z_hat) / s), 0, 2^q - 1) in float32; a constant group
  stores s = 1, code 0, z_hat = min;
* greedy: alpha_i = fp16(sum_l |r| / g) (float32 sum and divide), the residual
  update uses the stored fp16 alpha: r <- r - alpha_i b_i (one float32 rounding);
* alternating (a): G = B^T B is integer (exact), c = B^T w is a lane/butterfly
  float32 sum, alpha solves G alpha = c in float64 by Gaussian elimination
  without pivoting in row order (plain float64 operations, no fused
  multiply-add), stored as fp16; a pivot <= 0.5 (G singular: two planes equal
  or opposite) keeps the previous alpha for that group;
  (b) the 2^q levels v_k = sum_i (bit_i(k) ? +alpha_i : -alpha_i) accumulate
  in float32 in plane order; each element takes the k with the smallest
  |w - v_k| (float32), the lowest k on ties.
"""
from __future__ import annotations

import numpy as np

__all__ = ["quantize_rtn", "quantize_bcq_greedy", "quantize_bcq_alternating", "quantization_error",
           "lane_sum_f32"]

F32 = np.float32


def lane_sum_f32(v: np.ndarray) -> np.float32:
    """Sum of a float32 vector in the fixed lane/butterfly order (module header)."""
    v = np.asarray(v, dtype=F32)
    p = np.zeros(32, dtype=F32)
    for t in range(v.shape[0]):
        p[t % 32] = F32(p[t % 32] + v[t])
    idx = np.arange(32)
    for o in (16, 8, 4, 2, 1):
        p = (p + p[idx ^ o]).astype(F32)
    return p[0]


def _groups(n: int, g: int):
    return [(c0, min(n, c0 + g)) for c0 in range(0, n, g)]


def quantize_rtn(W: np.ndarray, q: int, g: int):
    """Uniform RTN: returns codes uint8 [m][n], scale fp16 [m][G], zero fp16 [m][G]
    with W ~ scale * code + zero per group (Eq. 6's additive z_hat, R16)."""
    W = np.asarray(W, dtype=np.float16)
    m, n = W.shape
    G = len(_groups(n, g))
    codes = np.zeros((m, n), dtype=np.uint8)
    scale = np.zeros((m, G), dtype=np.float16)
    zero = np.zeros((m, G), dtype=np.float16)
    top = F32(2 ** q - 1)
    for r in range(m):
        for k, (c0, c1) in enumerate(_groups(n, g)):
            w = W[r, c0:c1].astype(F32)
            mn, mx = w.min(), w.max()
            z16 = np.float16(mn)
            if mx == mn:
                s16 = np.float16(1.0)
                codes[r, c0:c1] = 0
            else:
                s16 = np.float16(F32(F32(mx - mn) / top))
                t = ((w - F32(z16)).astype(F32) / F32(s16)).astype(F32)
                codes[r, c0:c1] = np.clip(np.rint(t), 0, 2 ** q - 1).astype(np.uint8)
            scale[r, k], zero[r, k] = s16, z16
    return codes, scale, zero


def _pack_group_signs(planes: np.ndarray, r: int, c0: int, bits: np.ndarray, i: int):
    """Set plane i, row r, columns c0.. to the sign bits (1 = +1)."""
    for j, bit in enumerate(bits):
        c = c0 + j
        if bit:
            planes[i, r, c // 32] |= np.uint32(1) << np.uint32(c % 32)


def _greedy_group(w: np.ndarray, q: int):
    """Greedy residual fit of one group (float32 w); returns (alpha fp16 [q], signs bool [q][len])."""
    r = w.astype(F32).copy()
    gl = F32(w.shape[0])
    alpha = np.zeros(q, dtype=np.float16)
    signs = np.zeros((q, w.shape[0]), dtype=bool)
    for i in range(q):
        b = r >= 0
        a16 = np.float16(F32(lane_sum_f32(np.abs(r)) / gl))
        a = F32(a16)
        r = np.where(b, r - a, r + a).astype(F32)
        alpha[i], signs[i] = a16, b
    return alpha, signs


def quantize_bcq_greedy(W: np.ndarray, q: int, g: int):
    """Greedy BCQ: returns planes uint32 [q][m][ceil(n/32)], alpha fp16 [m][G][q]."""
    W = np.asarray(W, dtype=np.float16)
    m, n = W.shape
    grp = _groups(n, g)
    planes = np.zeros((q, m, (n + 31) // 32), dtype=np.uint32)
    alpha = np.zeros((m, len(grp), q), dtype=np.float16)
    for r in range(m):
        for k, (c0, c1) in enumerate(grp):
            a, s = _greedy_group(W[r, c0:c1].astype(F32), q)
            alpha[r, k] = a
            for i in range(q):
                _pack_group_signs(planes, r, c0, s[i], i)
    return planes, alpha


def _solve_alpha(signs: np.ndarray, w: np.ndarray, prev: np.ndarray) -> np.ndarray:
    """(a): least-squares alpha for fixed signs, as the header states; float64 result."""
    q = signs.shape[0]
    pm = np.where(signs, F32(1), F32(-1)).astype(F32)
    G = [[float(int(np.sum(signs[i] == signs[j])) * 2 - signs.shape[1]) for j in range(q)] for i in range(q)]
    c = [float(lane_sum_f32((pm[i] * w).astype(F32))) for i in range(q)]
    # Gaussian elimination without pivoting, row order, plain float64 ops
    A = [row[:] for row in G]
    bvec = c[:]
    for kk in range(q):
        piv = A[kk][kk]
        if not piv > 0.5:
            return prev.astype(np.float64)
        for i in range(kk + 1, q):
            f = A[i][kk] / piv
            for j in range(kk, q):
                A[i][j] = A[i][j] - f * A[kk][j]
            bvec[i] = bvec[i] - f * bvec[kk]
    x = [0.0] * q
    for i in range(q - 1, -1, -1):
        acc = bvec[i]
        for j in range(i + 1, q):
            acc = acc - A[i][j] * x[j]
        x[i] = acc / A[i][i]
    return np.array(x, dtype=np.float64)


def _nearest_signs(w: np.ndarray, alpha16: np.ndarray) -> np.ndarray:
    """(b): per element the pattern k whose level is nearest (lowest k on ties); signs [q][len]."""
    q = alpha16.shape[0]
    a = alpha16.astype(F32)
    K = 2 ** q
    v = np.zeros(K, dtype=F32)
    for k in range(K):
        acc = F32(0)
        for i in range(q):
            acc = F32(acc + (a[i] if (k >> i) & 1 else -a[i]))
        v[k] = acc
    err = np.abs((w[:, None] - v[None, :]).astype(F32))  # [len][K]
    best = np.argmin(err, axis=1)  # first minimum = lowest k
    return np.array([(best >> i) & 1 for i in range(q)], dtype=bool)


def quantize_bcq_alternating(W: np.ndarray, q: int, g: int, iters: int):
    """Greedy start, then `iters` rounds of (a) least-squares alpha, (b) nearest sign patterns."""
    W = np.asarray(W, dtype=np.float16)
    m, n = W.shape
    grp = _groups(n, g)
    planes = np.zeros((q, m, (n + 31) // 32), dtype=np.uint32)
    alpha = np.zeros((m, len(grp), q), dtype=np.float16)
    for r in range(m):
        for k, (c0, c1) in enumerate(grp):
            w = W[r, c0:c1].astype(F32)
            a16, s = _greedy_group(w, q)
            for _ in range(iters):
                a16 = _solve_alpha(s, w, a16.astype(np.float64)).astype(np.float16)
                s = _nearest_signs(w, a16)
            alpha[r, k] = a16
            for i in range(q):
                _pack_group_signs(planes, r, c0, s[i], i)
    return planes, alpha


def quantization_error(W: np.ndarray, W_hat: np.ndarray) -> dict:
    """mse, relative Frobenius error and max |error| of a reconstruction, float64."""
    W = np.asarray(W, dtype=np.float64)
    E = W - np.asarray(W_hat, dtype=np.float64)
    nw = np.linalg.norm(W)
    return {"mse": float(np.mean(E * E)), "rel_fro": float(np.linalg.norm(E) / nw) if nw else 0.0,
            "max_abs": float(np.max(np.abs(E))) if E.size else 0.0}
