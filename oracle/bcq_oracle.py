"""LUT-GEMM CPU oracle, fp64 -- TEST INFRASTRUCTURE ONLY.

This module is the plain, slow, obviously-correct definition of what the
LUT-GEMM hot path computes.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import it.
The product package ``paper_2206_09557_b200`` never imports it and shares no
code, header, table or constant generator with it; the CUDA path is checked
against it, never the other way round.

Citations: ``P:Lnnn`` is a line of the paper text (arXiv 2206.09557,
``PAPER.md``), with the section / equation named beside it.  ``R<k>`` names a
reading of an ambiguous passage, listed in DESIGN.md "Readings".

Canonical interchange layout (the bytes the GPU pack call also consumes):

* ``planes``  uint32 ``[q][m][ceil(n/32)]``: bit ``j`` of word ``w`` of row
  ``r`` of plane ``i`` is the binary weight b_i[r][32w+j]; bit 1 means +1 and
  bit 0 means -1 (R1: b = 2*b_hat - 1, App. C).  Padding bits beyond
  column n are ignored.
* ``alpha``   float16 ``[m][G][q]`` with ``G = ceil(n/g)``: scale alpha_i
  shared by the g consecutive columns of group ``c // g`` (Sec. 3.4,
  group-wise quantization; R7).
* ``offset``  float16 ``[m][G]`` or ``None``: the bias z of extended BCQ
  (Eq. 3), one per (row, group) (R5).
* ``X``       float16 ``[b][n]``: activations; ``Y`` is ``[b][m]`` (y = W x per
  batch row, Sec. 3.2).

All arithmetic is float64.  fp16 inputs convert to float64 exactly.

Pins: every function here is checked by ``tests/test_oracle_pins.py`` against
values the paper prints (Eq. 1 worked example, Table 5 sizes, the Sec. 4.1
"2.6x" count), closed forms, SPEC examples and brute force on tiny inputs.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "unpack_signs",
    "pack_signs",
    "dequantize",
    "bcq_gemv",
    "bcq_gemv_rows",
    "build_luts",
    "lut_keys",
    "lut_gemv",
    "uniform_dequantize",
    "uniform_to_bcq",
    "store_fp16",
    "memory_footprint_bits",
    "compression_ratio",
    "op_counts",
]


# ---------------------------------------------------------------------------
# Binary planes (Sec. 2.3: b_i in {-1,+1}^n; loaded as
# bits rather than "FP16 binary matrix" entries, R8)
# ---------------------------------------------------------------------------

def unpack_signs(planes: np.ndarray, n: int) -> np.ndarray:
    """Return the +-1 matrices b_i as int8 ``[q][rows][n]``.

    b_i[r][c] = 2 * bit(c mod 32 of word c // 32) - 1   (R1, R2).
    """
    planes = np.asarray(planes, dtype=np.uint32)
    cols = np.arange(n)
    words = planes[..., cols // 32]                       # [q][rows][n]
    bits = (words >> (cols % 32).astype(np.uint32)) & np.uint32(1)
    return (2 * bits.astype(np.int8) - 1).astype(np.int8)


def pack_signs(signs: np.ndarray) -> np.ndarray:
    """Inverse of :func:`unpack_signs`: +-1 ``[q][rows][n]`` -> uint32 words.

    Padding bits (columns >= n in the last word) are 0.
    """
    signs = np.asarray(signs)
    if not np.all((signs == 1) | (signs == -1)):
        raise ValueError("binary weights must be exactly +1 or -1")
    q, rows, n = signs.shape
    nw = (n + 31) // 32
    out = np.zeros((q, rows, nw), dtype=np.uint32)
    for c in range(n):
        bit = (signs[:, :, c] == 1).astype(np.uint32)
        out[:, :, c // 32] |= bit << np.uint32(c % 32)
    return out


# ---------------------------------------------------------------------------
# Extended BCQ reconstruction and the product it defines
# ---------------------------------------------------------------------------

def dequantize(planes, alpha, offset, n: int, g: int, rows=None) -> np.ndarray:
    """W_hat[r][c] = sum_i alpha[r][c//g][i] * b_i[r][c] + z[r][c//g].

    P:L258-261 Eq. 3 (extended BCQ, bias z); P:L296 (group-wise scales, R7);
    z per (row, group) (R5); z = 0 when ``offset is None``.
    Returns float64 ``[len(rows)][n]``.
    """
    planes = np.asarray(planes, dtype=np.uint32)
    if rows is None:
        rows = np.arange(planes.shape[1])
    rows = np.asarray(rows)
    signs = unpack_signs(planes[:, rows, :], n).astype(np.float64)   # [q][R][n]
    grp = np.arange(n) // g                                            # [n]
    a = np.asarray(alpha, dtype=np.float64)[rows][:, grp, :]           # [R][n][q]
    w = np.zeros((len(rows), n), dtype=np.float64)
    for i in range(planes.shape[0]):
        w += a[:, :, i] * signs[i]
    if offset is not None:
        w += np.asarray(offset, dtype=np.float64)[rows][:, grp]
    return w


def bcq_gemv_rows(planes, alpha, offset, X, n: int, g: int, rows) -> np.ndarray:
    """Y[beta][k] = sum_c W_hat[rows[k]][c] * X[beta][c], float64 ``[b][len(rows)]``.

    The definition of the LUT-GEMM product y = sum_i (A_i o (B_i x)) (P:L227
    Sec. 3.2) with the Eq. 3 bias added (R6): dequantise, then multiply.
    """
    x = np.atleast_2d(np.asarray(X, dtype=np.float64))
    w = dequantize(planes, alpha, offset, n, g, rows)
    return x @ w.T


def bcq_gemv(planes, alpha, offset, X, n: int, g: int, block_rows: int = 1024) -> np.ndarray:
    """Full product, row block by row block so memory stays bounded."""
    m = np.asarray(planes).shape[1]
    x = np.atleast_2d(np.asarray(X))
    y = np.empty((x.shape[0], m), dtype=np.float64)
    for r0 in range(0, m, block_rows):
        rows = np.arange(r0, min(m, r0 + block_rows))
        y[:, rows] = bcq_gemv_rows(planes, alpha, offset, x, n, g, rows)
    return y


# ---------------------------------------------------------------------------
# LUT formulation (Sec. 3.1; App. B)
# ---------------------------------------------------------------------------

def build_luts(x, mu: int = 8) -> np.ndarray:
    """T[t][k] = sum_{j<mu} (2*bit_j(k) - 1) * x[mu*t + j], x zero-padded.

    "pre-compute all possible combinations of full-precision activations and
    binary patterns" with sub-vector length mu.  Key bit j
    corresponds to column mu*t + j (LSB-first, R3).  float64 ``[ceil(n/mu)][2^mu]``.
    """
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    nt = (n + mu - 1) // mu
    xp = np.zeros(nt * mu, dtype=np.float64)
    xp[:n] = x
    keys = np.arange(2 ** mu)
    sign = np.empty((2 ** mu, mu), dtype=np.float64)
    for j in range(mu):
        sign[:, j] = 2.0 * ((keys >> j) & 1) - 1.0
    return xp.reshape(nt, mu) @ sign.T


def lut_keys(planes, n: int, mu: int = 8) -> np.ndarray:
    """key_i(r, t) = concatenation of the mu binary elements of row r of plane i
    in chunk t, LSB-first ("a key is given by concatenating mu binary
    elements"; R3).  int64 ``[q][rows][ceil(n/mu)]``; columns >= n give bit 0.
    """
    planes = np.asarray(planes, dtype=np.uint32)
    nt = (n + mu - 1) // mu
    cols = np.arange(nt * mu)
    valid = cols < n
    words = planes[..., np.minimum(cols, n - 1) // 32]
    bits = ((words >> (np.minimum(cols, n - 1) % 32).astype(np.uint32)) & np.uint32(1)).astype(np.int64)
    bits = bits * valid
    bits = bits.reshape(planes.shape[0], planes.shape[1], nt, mu)
    return (bits << np.arange(mu)).sum(axis=-1)


def lut_gemv(planes, alpha, offset, X, n: int, g: int, mu: int = 8, return_partials: bool = False):
    """LUT-form product, step by step in the paper's order.

    1. build one LUT per mu-chunk of x;
    2. partial dot products become retrievals: P[r][grp][i] = sum over the
       chunks t of group grp of T[t][key_i(r, t)];
    3. "those partial products are summed and then multiplied by scaling
       factors" (App. B): y_r = sum_grp sum_i alpha * P;
    4. bias term of Eq. 3 (R6): + z[r][grp] * sum_{c in grp} x_c.

    Requires ``g % mu == 0`` so no chunk straddles a group (R13).
    """
    if g % mu != 0:
        raise ValueError("LUT form needs g % mu == 0 (R13)")
    planes = np.asarray(planes, dtype=np.uint32)
    q, m, _ = planes.shape
    x2 = np.atleast_2d(np.asarray(X, dtype=np.float64))
    keys = lut_keys(planes, n, mu)                          # [q][m][nt]
    nt = keys.shape[-1]
    G = (n + g - 1) // g
    cpg = g // mu                                           # chunks per group
    a = np.asarray(alpha, dtype=np.float64)                 # [m][G][q]
    y = np.zeros((x2.shape[0], m), dtype=np.float64)
    partials = []
    for beta in range(x2.shape[0]):
        T = build_luts(x2[beta], mu)                        # [nt][2^mu]
        vals = T[np.arange(nt)[None, None, :], keys]        # [q][m][nt]
        P = np.zeros((m, G, q), dtype=np.float64)
        for t in range(nt):
            P[:, t // cpg, :] += vals[:, :, t].T
        partials.append(P)
        y[beta] = np.einsum("rgi,rgi->r", a, P)
        if offset is not None:
            xs = np.zeros(G, dtype=np.float64)
            for c in range(n):
                xs[c // g] += x2[beta, c]
            y[beta] += np.asarray(offset, dtype=np.float64) @ xs
    if return_partials:
        return y, partials
    return y


# ---------------------------------------------------------------------------
# Uniform quantization as extended BCQ (App. C)
# ---------------------------------------------------------------------------

def uniform_dequantize(codes, s, zhat, g: int) -> np.ndarray:
    """w_hat = s * sum_i 2^i * b_hat_i + z_hat = s * code + z_hat (Eq. 6).

    ``codes`` int ``[m][n]``; ``s``, ``zhat`` ``[m][G]``.  float64.
    """
    codes = np.asarray(codes, dtype=np.float64)
    n = codes.shape[1]
    grp = np.arange(n) // g
    return np.asarray(s, np.float64)[:, grp] * codes + np.asarray(zhat, np.float64)[:, grp]


def uniform_to_bcq(codes, s, zhat, q: int):
    """Convert uniform codes to extended BCQ exactly, in float64 (App. C).

    alpha_i = 2^(i-1) * s, b_i = 2 * b_hat_i - 1 with b_hat_i = bit i of the
    code, z = sum_i alpha_i + z_hat (Eq. 8 and the text after it;
    P:L620).  Plane index 0 is the least-significant bit (R4).

    Returns ``(planes uint32 [q][m][ceil(n/32)], alpha f64 [m][G][q], z f64 [m][G])``.
    """
    codes = np.asarray(codes, dtype=np.int64)
    if codes.min(initial=0) < 0 or codes.max(initial=0) >= 2 ** q:
        raise ValueError("codes must lie in [0, 2^q)")
    s = np.asarray(s, dtype=np.float64)
    zhat = np.asarray(zhat, dtype=np.float64)
    signs = np.stack([2 * ((codes >> i) & 1) - 1 for i in range(q)]).astype(np.int8)
    planes = pack_signs(signs)
    alpha = np.stack([s * 2.0 ** (i - 1) for i in range(q)], axis=-1)
    z = alpha.sum(axis=-1) + zhat
    return planes, alpha, z


def store_fp16(a):
    """Storage step: the kernel's scales/bias are FP16 ("A is an (m x 1)
    FP16 scaling matrix"; R12).  Round-to-nearest-even, as numpy's cast."""
    return np.asarray(a, dtype=np.float64).astype(np.float16)


# ---------------------------------------------------------------------------
# Closed-form models (Eq. 2, Eq. 4)
# ---------------------------------------------------------------------------

def memory_footprint_bits(m: int, n: int, q: int, g: int, scales_per_group: int | None = None,
                          bias: bool = False) -> dict:
    """S = S_b + S_alpha, S_b = m*n*q bits, S_alpha = 16*m*(n/g)*q bits
    (Eq. 4).  ``scales_per_group`` defaults to q (Eq. 4's count); a
    uniform-converted tensor needs only 1 (alpha_i = 2^(i-1) s, R18, Table 5).
    A bias adds 16 bits per (row, group)."""
    spg = q if scales_per_group is None else scales_per_group
    G = (n + g - 1) // g
    s_b = m * n * q
    s_a = 16 * m * G * spg
    s_z = 16 * m * G if bias else 0
    return {"S_b": s_b, "S_alpha": s_a, "S_z": s_z, "S": s_b + s_a + s_z}


def compression_ratio(m: int, n: int, q: int, g: int, scales_per_group: int | None = None,
                      bias: bool = False) -> float:
    """16-bit dense size over the quantized size (Table 5 "Comp. Ratio")."""
    fp = memory_footprint_bits(m, n, q, g, scales_per_group, bias)
    return 16.0 * m * n / fp["S"]


def op_counts(m: int, n: int, q: int, mu: int = 8) -> dict:
    """C_build = 2^mu * n/mu, C_read = m * n/mu * q (Eq. 2), against
    the m*n multiply-accumulates of a dense product."""
    nt = (n + mu - 1) // mu
    return {"c_build": (2 ** mu) * nt, "c_read": m * nt * q, "dense_macs": m * n}
