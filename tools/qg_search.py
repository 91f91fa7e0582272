"""q x g trade-off explorer (App. D-E): for one dense fp16 layer, quantize
with the GPU quantizers for every (q, g), and report reconstruction error (relative
Frobenius, the stand-in for the paper's LAMBADA accuracy, which needs trained
weights), compression vs fp16 (Eq. 4 bytes actually stored) and the measured
LUT-GEMV latency -- the search space Fig. 4(b) / Fig. 7 explore.

    python tools/qg_search.py [--m 12288] [--n 12288] [--method bcq|alt|rtn] [--iters 2]

The weight is seeded Gaussian with per-row scale variation (or --npy a [m][n] file).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2206_09557_b200 as L  # noqa: E402


def dequant_bcq(planes, alpha, n, g):
    """Device reconstruction sum_i alpha_i b_i (test tool only; not a product path)."""
    q, m, nw = planes.shape
    bits = ((planes.view(torch.int32).unsqueeze(-1) >> torch.arange(32, device=planes.device)) & 1).reshape(q, m, nw * 32)
    sgn = bits.float() * 2 - 1
    a = alpha.float().repeat_interleave(g, dim=1)  # [m][n][q]
    return (sgn.permute(1, 2, 0) * a).sum(-1)


def time_gemv(w, n, reps=200):
    x = torch.randn(n, device="cuda").half()
    y = torch.empty(w.m, device="cuda", dtype=torch.float16)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(w.m, n, 1), "cuda")
    for _ in range(5):
        L.lutgemm_gemv(w, x, y, ws)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            L.lutgemm_gemv(w, x, y, ws)
    g.replay()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps // 20):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / reps * 1e3  # us (L2-warm: one weight copy)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=12288)
    ap.add_argument("--n", type=int, default=12288)
    ap.add_argument("--method", default="alt", choices=["bcq", "alt", "rtn"])
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--npy", default="")
    a = ap.parse_args()
    torch.manual_seed(0)
    if a.npy:
        W = torch.from_numpy(np.load(a.npy)).half().cuda()
    else:
        W = (torch.randn(a.m, a.n, device="cuda") * (0.5 + torch.rand(a.m, 1, device="cuda")) * 0.02).half()
    m, n = W.shape
    Wf = W.float()
    for q in (1, 2, 3, 4):
        for g in (32, 64, 128, 256, n):
            if a.method == "rtn":
                c, s, z = L.lutgemm_quantize_rtn(W, q, g)
                w = L.lutgemm_pack_uniform(c, s, z, q, g, compact=True)
                Wh = (s.float().repeat_interleave(g, 1) * c.float() + z.float().repeat_interleave(g, 1))
            else:
                planes, alpha = L.lutgemm_quantize_bcq(W, q, g, 0 if a.method == "bcq" else a.iters)
                w = L.lutgemm_pack_bcq(planes, alpha, None, n, g)
                Wh = dequant_bcq(planes, alpha, n, g)
            err = float(torch.linalg.norm(Wf - Wh) / torch.linalg.norm(Wf))
            us = time_gemv(w, n)
            print(json.dumps({"method": a.method, "q": q, "g": g, "rel_fro": round(err, 5),
                              "compression_vs_fp16": round(2 * m * n / w.nbytes(), 2), "packed_MB": round(w.nbytes() / 1e6, 2),
                              "gemv_us_l2_warm": round(us, 2)}), flush=True)
            del w, Wh
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
