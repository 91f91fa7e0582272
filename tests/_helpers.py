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
    """Independent statement of layout.cuh: slice s = 1024 columns, L_s lanes
    (32 columns each), row quads; planes[s][rq][i][lane][r4] uint32,
    alpha[rq][i][G][r4], offset[rq][G][r4]; padded rows are zero."""
    m4 = (m + 3) // 4 * 4
    RQ = m4 // 4
    G = n // g
    nw = n // 32
    P = np.zeros((q, m4, nw), dtype=np.uint32)
    P[:, :m] = planes
    out = []
    for s in range((n + 1023) // 1024):
        w0, w1 = 32 * s, min(nw, 32 * s + 32)
        blk = P[:, :, w0:w1]                                   # [q][m4][L]
        blk = blk.reshape(q, RQ, 4, w1 - w0).transpose(1, 0, 3, 2)   # [RQ][q][L][4]
        out.append(np.ascontiguousarray(blk).reshape(-1))
    planes_native = np.concatenate(out).view(np.uint8)
    A = np.zeros((m4, G, q), dtype=np.float16)
    A[:m] = alpha
    alpha_native = A.reshape(RQ, 4, G, q).transpose(0, 3, 2, 1).reshape(-1)
    off_native = None
    if offset is not None:
        Z = np.zeros((m4, G), dtype=np.float16)
        Z[:m] = offset
        off_native = Z.reshape(RQ, 4, G).transpose(0, 2, 1).reshape(-1)
    return planes_native, alpha_native, off_native
