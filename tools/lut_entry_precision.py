"""NEXT-3 precision study: can the LUT entries be narrower than fp32?

A 2-byte entry halves the shared-memory bytes per lookup, i.e. the batched
roof, so the question is whether the product still meets
north_star's tolerances (rel-L2 <= 2e-3 and max elementwise rel <= 1e-2 with
the R22 floor max(|y|, 1e-3 rms(y))).  This simulates the LUT formulation
exactly in numpy on a row sample of fc1 (n = 12288, q = 3, g = 128, the
BASELINE input recipe), with the table entries T_t[k] = sum_j (2 bit_j(k) - 1)
x_j stored as:

  fp32        the shipped kernels (exact: a sum of 8 fp16 values fits 24 bits here)
  fp16        round-to-nearest-even fp16 entries
  bf16        round-to-nearest-even bf16 entries
  int16/tab   16-bit fixed point with one power-of-two scale per table (chunk)
  fp16x2      a compensated pair hi = fp16(T), lo = fp16(T - hi) (4 bytes again)

The accumulation is fp32 in every case (per (row, group, plane) partial sums,
scaled by the fp16 alpha, as the kernels do), and the result is compared with
the exact fp64 product.  Standalone: no import of the product package or of
oracle/ (this is an analysis tool, not a test).

    python tools/lut_entry_precision.py [--rows 1024] [--batch 4]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workloads import gen_bcq, gen_x  # noqa: E402


def signs_table() -> np.ndarray:
    k = np.arange(256)[:, None]
    return (2.0 * ((k >> np.arange(8)[None, :]) & 1) - 1.0)  # [256][8]


def store(T: np.ndarray, kind: str) -> np.ndarray:
    """T float64 [chunks][256] -> the stored entry value (float64)."""
    if kind == "fp32":
        return T.astype(np.float32).astype(np.float64)
    if kind == "fp16":
        return T.astype(np.float16).astype(np.float64)
    if kind == "bf16":
        u = T.astype(np.float32).view(np.uint32).astype(np.uint64)
        r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        return r.astype(np.uint32).view(np.float32).astype(np.float64)
    if kind == "int16/tab":
        amax = np.max(np.abs(T), axis=1, keepdims=True)
        e = np.ceil(np.log2(np.maximum(amax, 1e-30) / 32767.0))
        sc = 2.0 ** e
        return np.clip(np.rint(T / sc), -32768, 32767) * sc
    if kind == "fp16x2":
        hi = T.astype(np.float16).astype(np.float64)
        lo = (T - hi).astype(np.float16).astype(np.float64)
        return hi + lo
    raise ValueError(kind)


def lut_product(planes, alpha, X, n, g, kind):
    """y[b][r] = sum_grp sum_i alpha[r][grp][i] * fp32(sum_{t in grp} Tstored_t[key_i(r, t)])."""
    q, m, _ = planes.shape
    S = signs_table()
    nchunks = n // 8
    keys = planes.view(np.uint8).reshape(q, m, -1)[:, :, :nchunks].astype(np.int64)  # byte t = key of chunk t
    Y = np.zeros((X.shape[0], m))
    for b in range(X.shape[0]):
        x = X[b].astype(np.float64).reshape(nchunks, 8)
        T = store(x @ S.T, kind)                                      # [chunks][256]
        looked = T[np.arange(nchunks)[None, None, :], keys]           # [q][m][chunks]
        G = n // g
        part = looked.reshape(q, m, G, g // 8).astype(np.float32).sum(axis=3, dtype=np.float32)  # fp32 partials
        Y[b] = np.einsum("imk,mki->m", part.astype(np.float64), alpha.astype(np.float64))
    return Y


def exact_product(planes, alpha, X, n, g):
    q, m, _ = planes.shape
    bits = np.unpackbits(planes.view(np.uint8).reshape(q, m, -1), axis=2, bitorder="little")[:, :, :n]
    W = np.zeros((m, n))
    grp = np.arange(n) // g
    for i in range(q):
        W += alpha[:, grp, i].astype(np.float64) * (2.0 * bits[i] - 1.0)
    return X.astype(np.float64) @ W.T


def metrics(y, ref):
    err = y - ref
    rms = math.sqrt(float(np.mean(ref ** 2)))
    return {"rel_l2": float(np.linalg.norm(err) / np.linalg.norm(ref)),
            "max_rel_floored": float(np.max(np.abs(err) / np.maximum(np.abs(ref), 1e-3 * rms))),
            "max_rel_raw": float(np.max(np.abs(err) / np.abs(ref)))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=4)
    a = ap.parse_args()
    m, n, q, g = a.rows, 12288, 3, 128
    d = gen_bcq(2206, m, n, q, g)
    X = gen_x(9557, a.batch, n)
    ref = exact_product(d["planes"], d["alpha"], X, n, g)
    for kind in ("fp32", "fp16", "bf16", "int16/tab", "fp16x2"):
        r = metrics(lut_product(d["planes"], d["alpha"], X, n, g, kind), ref)
        r.update(entry=kind, bytes_per_entry=4 if kind in ("fp32", "fp16x2") else 2, rows=m, batch=a.batch,
                 shape="fc1 rows (n=12288, q=3, g=128)",
                 passes=bool(r["rel_l2"] <= 2e-3 and r["max_rel_floored"] <= 1e-2))
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
