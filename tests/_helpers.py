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
    L_s lanes of 32 columns); slice s = three regions, each zero-padded to a
    multiple of 256 bytes: keys [RQ][q][L_s][4 rows] uint32, alpha
    [RQ][gps][q][4 rows] fp16, z [RQ][gps][4 rows] fp16 (if offset);
    gps = 32 L_s / g (g <= 1024) else 1."""
    m4 = (m + 3) // 4 * 4
    RQ = m4 // 4
    G = n // g
    nw = n // 32
    P = np.zeros((q, m4, nw), dtype=np.uint32)
    P[:, :m] = planes
    A = np.zeros((m4, G, q), dtype=np.float16)
    A[:m] = alpha
    Z = np.zeros((m4, G), dtype=np.float16)
    if offset is not None:
        Z[:m] = offset

    def pad256(b):
        return np.concatenate([b, np.zeros((-len(b)) % 256, np.uint8)])

    out = []
    for s in range((n + 1023) // 1024):
        w0, w1 = 32 * s, min(nw, 32 * s + 32)
        L = w1 - w0
        if g <= 1024:
            gps = 32 * L // g
            grps = list(range(s * (1024 // g), s * (1024 // g) + gps))
        else:
            gps, grps = 1, [(s * 1024) // g]
        keys = P[:, :, w0:w1].reshape(q, RQ, 4, L).transpose(1, 0, 3, 2)          # [RQ][q][L][4]
        al = A[:, grps, :].reshape(RQ, 4, gps, q).transpose(0, 2, 3, 1)           # [RQ][gps][q][4]
        out.append(pad256(np.ascontiguousarray(keys).view(np.uint8).reshape(-1)))
        out.append(pad256(np.ascontiguousarray(al).view(np.uint8).reshape(-1)))
        if offset is not None:
            zz = Z[:, grps].reshape(RQ, 4, gps).transpose(0, 2, 1)                 # [RQ][gps][4]
            out.append(pad256(np.ascontiguousarray(zz).view(np.uint8).reshape(-1)))
    return np.concatenate(out)
