"""Test helpers: parity metrics (north_star tolerances) and an independent
numpy re-statement of the kernel-native layout (DESIGN.md "Data layout in
HBM") used to check the GPU packer byte for byte."""
from __future__ import annotations

import numpy as np

REL_L2_TOL = 2e-3          # north_star: relative L2 error <= 2e-3
MAX_REL_TOL = 1e-2         # north_star: max elementwise relative error <= 1e-2
FLOOR = 1e-3               # R22: denominator max(|y|, 1e-3 * rms(y))


def parity(y_gpu, y_ref) -> dict:
    y_gpu = np.asarray(y_gpu, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    err = y_gpu - y_ref
    rms = np.sqrt(np.mean(y_ref ** 2))
    rel_l2 = float(np.linalg.norm(err) / max(np.linalg.norm(y_ref), 1e-300))
    max_rel = float(np.max(np.abs(err) / np.maximum(np.abs(y_ref), FLOOR * rms)))
    raw = float(np.max(np.abs(err) / np.maximum(np.abs(y_ref), 1e-300)))
    return {"rel_l2": rel_l2, "max_rel": max_rel, "max_rel_unfloored": raw}


def assert_parity(y_gpu, y_ref, what=""):
    p = parity(y_gpu, y_ref)
    assert p["rel_l2"] <= REL_L2_TOL and p["max_rel"] <= MAX_REL_TOL, f"{what}: {p}"
    return p


def native_pack_reference(planes: np.ndarray, alpha: np.ndarray, offset, m: int, n: int, q: int, g: int):
    """Independent statement of layout.cuh: slice-major (1024 columns per slice,
    L_s lanes of 32 columns, the last lane possibly partial); slice s = three
    regions, each zero-padded to a multiple of 256 bytes: keys [RQ][q][L_s][4 rows]
    uint32, alpha [RQ][gps][q][4 rows] fp16, z [RQ][gps][4 rows] fp16 (if offset).
    Scale entries per slice (gps) by group class:
      g == n or a multiple of 1024: 1 entry, the group holding the slice's first column;
      g | 1024 (g % 32 == 0): 32 L_s / g groups;
      other g % 32 == 0: (g + 991) // g + 1 entries, groups floor(1024 s / g) + k
        (entries past the last group are zero);
      g % 32 != 0 (chunk groups): alpha [RQ][L_s][q][4 chunks][4 rows] and
        z [RQ][L_s][4 chunks][4 rows], entry (lane p, chunk j) = group of column
        1024 s + 32 p + 8 j (zero past n)."""
    m4 = (m + 3) // 4 * 4
    RQ = m4 // 4
    G = n // g
    nw = (n + 31) // 32
    P = np.zeros((q, m4, nw), dtype=np.uint32)
    P[:, :m] = planes
    A = np.zeros((m4, G + 1, q), dtype=np.float16)   # group index G = the zero entry
    A[:m, :G] = alpha
    Z = np.zeros((m4, G + 1), dtype=np.float16)
    if offset is not None:
        Z[:m, :G] = offset

    def pad256(b):
        return np.concatenate([b, np.zeros((-len(b)) % 256, np.uint8)])

    chunk = g % 32 != 0 and g != n
    out = []
    for s in range((n + 1023) // 1024):
        w0, w1 = 32 * s, min(nw, 32 * s + 32)
        L = w1 - w0
        keys = P[:, :, w0:w1].reshape(q, RQ, 4, L).transpose(1, 0, 3, 2)          # [RQ][q][L][4]
        out.append(pad256(np.ascontiguousarray(keys).view(np.uint8).reshape(-1)))
        if chunk:
            cols = 1024 * s + 32 * np.arange(L)[:, None] + 8 * np.arange(4)[None, :]  # [L][4]
            grp = np.where(cols < n, cols // g, G)
            al = A[:, grp.reshape(-1), :].reshape(RQ, 4, L, 4, q).transpose(0, 2, 4, 3, 1)  # [RQ][L][q][4][4]
            zz = Z[:, grp.reshape(-1)].reshape(RQ, 4, L, 4).transpose(0, 2, 3, 1)           # [RQ][L][4][4]
        else:
            if g == n or (g >= 1024 and g % 1024 == 0):
                grps = [(s * 1024) // g]
            elif 1024 % g == 0:
                grps = list(range(s * (1024 // g), s * (1024 // g) + 32 * L // g))
            else:
                grps = [min(G, (s * 1024) // g + k) for k in range((g + 991) // g + 1)]
            gps = len(grps)
            al = A[:, grps, :].reshape(RQ, 4, gps, q).transpose(0, 2, 3, 1)       # [RQ][gps][q][4]
            zz = Z[:, grps].reshape(RQ, 4, gps).transpose(0, 2, 1)                 # [RQ][gps][4]
        out.append(pad256(np.ascontiguousarray(al).view(np.uint8).reshape(-1)))
        if offset is not None:
            out.append(pad256(np.ascontiguousarray(zz).view(np.uint8).reshape(-1)))
    return np.concatenate(out)


# ---------------------------------------------------------------------------
# quantizer tie rule (RQ5): GPU quantizer outputs vs the plain fp64 oracle
# (oracle/quantize_plain.py), which flags every (row, group) with a decision inside
# the float32 error the kernel may make
# ---------------------------------------------------------------------------

def _group_cols(n, g):
    return [(c0, min(n, c0 + g)) for c0 in range(0, n, g)]


def check_rtn_rule(got, ref, fragile, W, q, g, cap):
    """got/ref = (codes, scale, zero).  Non-fragile groups bit-equal; fragile share <= cap; a
    fragile group's max reconstruction error within one level s of the oracle's."""
    gc, gs, gz = (np.asarray(a) for a in got)
    rc, rs, rz = ref
    m, n = gc.shape
    W = np.asarray(W, dtype=np.float64)
    nfr = 0
    for r in range(m):
        for k, (c0, c1) in enumerate(_group_cols(n, g)):
            if fragile[r, k]:
                nfr += 1
                eg = np.abs(W[r, c0:c1] - (float(gs[r, k]) * gc[r, c0:c1] + float(gz[r, k]))).max()
                er = np.abs(W[r, c0:c1] - (float(rs[r, k]) * rc[r, c0:c1] + float(rz[r, k]))).max()
                assert eg <= er + float(rs[r, k]) * 1.01, (r, k, eg, er)
                continue
            assert gs[r, k].view(np.uint16) == rs[r, k].view(np.uint16), ("s", r, k, gs[r, k], rs[r, k])
            assert gz[r, k].view(np.uint16) == rz[r, k].view(np.uint16), ("z", r, k)
            assert np.array_equal(gc[r, c0:c1], rc[r, c0:c1]), ("codes", r, k)
    share = nfr / fragile.size
    assert share <= cap, f"fragile share {share:.4f} > {cap}"
    return share


def check_bcq_rule(got, ref, fragile, W, q, g, cap, rel_slack=0.05):
    """got/ref = (planes, alpha).  Non-fragile groups: alpha bits and signs equal; fragile share
    <= cap; a fragile group's reconstruction error within (1 + rel_slack) of the oracle's."""
    from oracle import dequantize, unpack_signs
    gp, ga = (np.asarray(a) for a in got)
    rp, ra = ref
    m, n = W.shape
    W = np.asarray(W, dtype=np.float64)
    gsg = unpack_signs(gp.view(np.uint32), n)
    rsg = unpack_signs(rp.view(np.uint32), n)
    Wg = dequantize(gp.view(np.uint32), ga, None, n, g)
    Wr = dequantize(rp.view(np.uint32), ra, None, n, g)
    nfr = 0
    for r in range(m):
        for k, (c0, c1) in enumerate(_group_cols(n, g)):
            if fragile[r, k]:
                nfr += 1
                eg = np.linalg.norm(W[r, c0:c1] - Wg[r, c0:c1])
                er = np.linalg.norm(W[r, c0:c1] - Wr[r, c0:c1])
                assert eg <= er * (1 + rel_slack) + 1e-3 * np.linalg.norm(W[r, c0:c1]) + 1e-12, (r, k, eg, er)
                continue
            assert np.array_equal(ga[r, k].view(np.uint16), ra[r, k].view(np.uint16)), ("alpha", r, k, ga[r, k],
                                                                                         ra[r, k])
            assert np.array_equal(gsg[:, r, c0:c1], rsg[:, r, c0:c1]), ("signs", r, k)
    share = nfr / fragile.size
    assert share <= cap, f"fragile share {share:.4f} > {cap}"
    return share


# ---------------------------------------------------------------------------
# full-size oracle runs: row blocks of oracle.bcq_gemv_rows in worker processes
# (test infrastructure only; the arithmetic is the oracle's, unchanged)
# ---------------------------------------------------------------------------

_POOL_ARGS = None


def _oracle_block(rows):
    import oracle as O
    planes, alpha, offset, X, n, g = _POOL_ARGS
    return O.bcq_gemv_rows(planes, alpha, offset, X, n, g, rows)


def oracle_rows_parallel(planes, alpha, offset, X, n, g, rows=None, block=512, procs=None):
    """oracle.bcq_gemv_rows over `rows` (default: all), split into row blocks evaluated by
    forked worker processes (numpy only in the children).  float64 [b][len(rows)]."""
    import multiprocessing as mp
    import os
    global _POOL_ARGS
    m = np.asarray(planes).shape[1]
    rows = np.arange(m) if rows is None else np.asarray(rows)
    blocks = [rows[i:i + block] for i in range(0, len(rows), block)]
    _POOL_ARGS = (planes, alpha, offset, np.atleast_2d(X), n, g)
    procs = procs or min(len(blocks), max(1, (os.cpu_count() or 2) - 1), 16)
    try:
        if procs <= 1:
            parts = [_oracle_block(b) for b in blocks]
        else:
            with mp.get_context("fork").Pool(procs) as pool:
                parts = pool.map(_oracle_block, blocks)
    finally:
        _POOL_ARGS = None
    return np.concatenate(parts, axis=1)


def stratified_rows(m, per_block=2, block=256, seed=0):
    """Rows sampled from EVERY block of `block` consecutive rows (so every reducer range of the
    fused cross-slice reduction is checked), plus the first and last rows."""
    rng = np.random.default_rng(seed)
    rows = set()
    for b0 in range(0, m, block):
        b1 = min(m, b0 + block)
        rows.update(rng.choice(np.arange(b0, b1), size=min(per_block, b1 - b0), replace=False).tolist())
    rows |= {0, 1, 2, 3, m - 4, m - 3, m - 2, m - 1}
    return np.array(sorted(r for r in rows if 0 <= r < m))
