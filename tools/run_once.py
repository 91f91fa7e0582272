"""Run one LUT-GEMM product shape a few times eagerly (for ncu captures).

    python tools/run_once.py M N Q G [B] [--uniform] [--iters K]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import gen_bcq, gen_uniform, gen_x  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", type=int, nargs="+")
    ap.add_argument("--uniform", action="store_true")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    m, n, q, g = a.shape[:4]
    b = a.shape[4] if len(a.shape) > 4 else 1
    dev = torch.device("cuda")
    if a.uniform:
        u = gen_uniform(7, m, n, q, g)
        w = L.lutgemm_pack_uniform(*(torch.from_numpy(u[k]).to(dev) for k in ("codes", "scale", "zero")), q, g)
    else:
        d = gen_bcq(7, m, n, q, g)
        w = L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).to(dev),
                               torch.from_numpy(d["alpha"]).to(dev), None, n, g)
    X = torch.from_numpy(gen_x(7, b, n)).to(dev)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(m, n, b), dev)
    for _ in range(a.iters):
        if b == 1:
            L.lutgemm_gemv(w, X[0], None, ws)
        else:
            L.lutgemm_gemm_batched(w, X, None, ws)
    torch.cuda.synchronize()
    print("ok", m, n, q, g, b)


if __name__ == "__main__":
    main()
