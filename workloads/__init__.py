"""Seeded synthetic inputs for LUT-GEMM -- shared by tests, bench and smoke.

This module holds NO arithmetic of the method: it only draws random bits,
scales, codes and activations with the shapes and distributions of the
paper's workloads.  Both the CUDA path and the CPU
oracle consume what it returns; neither is imported here.

Shape convention: W is m x n (m output rows, n reduction columns), y = W x
(P:L202).  BASELINE.json writes "in x out", so "12288x49152" is
OPT-175B fc1 with n=12288, m=49152.
"""
from __future__ import annotations

import math

import numpy as np

# BASELINE.json configs, restated as (m, n, q, g, b, offset).
CONFIGS = {
    "tiny": dict(m=512, n=512, q=3, g=128, b=1, seed=101),
    "attn": dict(m=12288, n=12288, q=3, g=128, b=1, seed=2),
    "fc1": dict(m=49152, n=12288, q=3, g=128, b=1, seed=301),
    "fc2": dict(m=12288, n=49152, q=3, g=128, b=1, seed=302),
    "llama_sq": dict(m=8192, n=8192, q=4, g=128, b=1, seed=401, uniform=True),
    "llama_up": dict(m=22016, n=8192, q=4, g=128, b=1, seed=402, uniform=True),
    "llama_down": dict(m=8192, n=22016, q=4, g=128, b=1, seed=403, uniform=True),
}

# OPT-175B decoder linears per layer (BASELINE config 5): (name, m, n).
OPT175B_LINEARS = [("qkv", 36864, 12288), ("out", 12288, 12288),
                   ("fc1", 49152, 12288), ("fc2", 12288, 49152)]


def _rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def random_planes(rng: np.random.Generator, q: int, m: int, n: int) -> np.ndarray:
    """Uniform random bits in the canonical uint32 ``[q][m][ceil(n/32)]`` layout
    (every mu=8 key uniform on 0..255); padding bits beyond n are zero."""
    nw = (n + 31) // 32
    words = rng.integers(0, 1 << 32, size=(q, m, nw), dtype=np.uint64).astype(np.uint32)
    if n % 32:
        words[:, :, -1] &= np.uint32((1 << (n % 32)) - 1)
    return words


def gen_bcq(seed: int, m: int, n: int, q: int, g: int, offset: bool = False) -> dict:
    """Non-uniform BCQ weights (configs 1, 2, 3, 5).

    alpha[r][grp][i] = fp16(0.87 * 2^-i * U(0.75, 1.25) / sqrt(n)) so that the
    planes carry decreasing weight like a greedy BCQ fit; z ~ fp16(0.1 N(0,1)/sqrt(n))
    when an offset is requested.
    """
    rng = _rng(seed)
    G = (n + g - 1) // g
    planes = random_planes(rng, q, m, n)
    u = rng.uniform(0.75, 1.25, size=(m, G, q))
    alpha = (0.87 * (2.0 ** -np.arange(q)) * u / math.sqrt(n)).astype(np.float16)
    z = None
    if offset:
        z = (0.1 * rng.standard_normal((m, G)) / math.sqrt(n)).astype(np.float16)
    return {"m": m, "n": n, "q": q, "g": g, "planes": planes, "alpha": alpha, "offset": z}


def gen_uniform(seed: int, m: int, n: int, q: int, g: int) -> dict:
    """Uniformly quantized weights (config 4, LLaMA shapes, AWQ-style).

    codes ~ U{0..2^q-1} (uint8 ``[m][n]``); s = fp16(U(0.5, 1.5) / (8 sqrt(n)))
    (kept >= 2^-13 so s/2 is a normal fp16); integer zero-point zp ~ U{0..2^q-1}
    expressed as the additive z_hat = fp16(-s * zp) of Eq. 6 (R16).
    """
    rng = _rng(seed)
    G = (n + g - 1) // g
    codes = rng.integers(0, 2 ** q, size=(m, n), dtype=np.uint8)
    s = (rng.uniform(0.5, 1.5, size=(m, G)) / (8.0 * math.sqrt(n))).astype(np.float16)
    zp = rng.integers(0, 2 ** q, size=(m, G))
    zhat = (-(s.astype(np.float64)) * zp).astype(np.float16)
    return {"m": m, "n": n, "q": q, "g": g, "codes": codes, "scale": s, "zero": zhat}


def gen_x(seed: int, b: int, n: int) -> np.ndarray:
    """Activations x ~ N(0, 1), fp16 ``[b][n]``."""
    return _rng(seed + 7919).standard_normal((b, n)).astype(np.float16)
