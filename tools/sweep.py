"""Measure the LUT-GEMM path on the other BASELINE.json configs (parity-tested
shapes): attention 12288^2 q x g grid, fc1/fc2, LLaMA-65B uniform shapes with
offset, and batched fc1/fc2 b = 1..32.  One JSON line per case on stdout.

    python tools/sweep.py [--only attn,ffn,llama,batched] [--steps 400]

Timing as in bench.py: CUDA graph of consecutive products on rotating weight
copies (> 3x L2), events around the replays.  The roofline line for b = 1 is
HBM (B_alg / time); for b >= 2 the shared-memory lookup rate is reported too:
lookups/32 warp-LDS per SM at 1 wavefront per cycle.
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
from bench import algorithmic_bytes, measured_peaks  # noqa: E402
from workloads import gen_bcq, gen_uniform, gen_x  # noqa: E402

SM_HZ = 1.965e9


def time_product(ws_list, X, b, m, n, steps):
    dev = X.device
    Y = torch.empty((b, m), dtype=torch.float16, device=dev)
    wsb = L.make_workspace(L.lutgemm_workspace_bytes(m, n, b), dev)

    def step(i):
        w = ws_list[i % len(ws_list)]
        if b == 1:
            L.lutgemm_gemv(w, X[0], Y[0], wsb)
        else:
            L.lutgemm_gemm_batched(w, X, Y, wsb)

    for i in range(4):
        step(i)
    torch.cuda.synchronize()
    G = max(len(ws_list), min(steps, 40) // len(ws_list) * len(ws_list))
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=cap):
        for i in range(G):
            step(i)
    graph.replay()
    torch.cuda.synchronize()
    reps = max(1, math.ceil(steps / G))
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        graph.replay()
    e.record()
    torch.cuda.synchronize()
    chain = a.elapsed_time(e) / (reps * G) * 1e3  # us per product in the graph chain
    # isolated: events around each eager launch (no overlap with a neighbour)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(40)]
    for i, (e0, e1) in enumerate(ev):
        e0.record()
        step(i)
        e1.record()
    torch.cuda.synchronize()
    iso = float(np.median([e0.elapsed_time(e1) for e0, e1 in ev])) * 1e3
    return chain, iso


def case(name, m, n, q, g, b=1, uniform=False, steps=400, seed=7, compact=False):
    dev = torch.device("cuda")
    offset = uniform
    B = algorithmic_bytes(m, n, q, g, b, offset, compact)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    ncopies = max(2, math.ceil(3 * l2 / B))
    if uniform:
        u = gen_uniform(seed, m, n, q, g)
        codes, s, z = (torch.from_numpy(u[k]).to(dev) for k in ("codes", "scale", "zero"))
        ws_list = [L.lutgemm_pack_uniform(codes, s, z, q, g, compact=compact) for _ in range(ncopies)]
    else:
        d = gen_bcq(seed, m, n, q, g)
        planes = torch.from_numpy(d["planes"].view(np.int32)).to(dev)
        alpha = torch.from_numpy(d["alpha"]).to(dev)
        ws_list = [L.lutgemm_pack_bcq(planes, alpha, None, n, g) for _ in range(ncopies)]
    X = torch.from_numpy(gen_x(seed, b, n)).to(dev)
    us, iso = time_product(ws_list, X, b, m, n, steps)
    peak = measured_peaks()["hbm_gbs"]
    gbs = B / (us * 1e-6) / 1e9
    lookups = m * q * (n // 8) * b
    lds_us = lookups / 32 / torch.cuda.get_device_properties(dev).multi_processor_count / SM_HZ * 1e6
    hbm_us = B / (peak * 1e9) * 1e6
    out = {"case": name, "m": m, "n": n, "q": q, "g": g, "b": b, "offset": offset, "compact": compact,
           "us": round(us, 3), "iso_us": round(iso, 3), "frac_hbm_iso": round(B / (iso * 1e-6) / 1e9 / measured_peaks()["hbm_gbs"], 4),
           "GBps": round(gbs, 1), "frac_hbm": round(gbs / peak, 4), "bytes_alg": B,
           "hbm_roof_us": round(hbm_us, 2), "lds_roof_us": round(lds_us, 2),
           "bound": "hbm" if hbm_us >= lds_us else "lds",
           "frac_of_binding_roof": round(max(hbm_us, lds_us) / us, 4)}
    print(json.dumps(out), flush=True)
    del ws_list
    torch.cuda.empty_cache()
    return out


def dense_fp16(m, n, b, steps=200):
    """Context only (a comparison system): cuBLAS fp16 Y = X W^T on a
    dense fp16 weight of the same shape, rotating copies > 3x L2, graph-timed."""
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    nc = max(2, math.ceil(3 * l2 / (2 * m * n)))
    Ws = [torch.randn(m, n, device=dev, dtype=torch.float16) * 0.01 for _ in range(nc)]
    X = torch.randn(b, n, device=dev, dtype=torch.float16)
    Y = torch.empty(b, m, device=dev, dtype=torch.float16)
    for i in range(3):
        torch.matmul(X, Ws[i % nc].t(), out=Y)
    torch.cuda.synchronize()
    G = nc * max(1, 20 // nc)
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cap):
        for i in range(G):
            torch.matmul(X, Ws[i % nc].t(), out=Y)
    g.replay()
    torch.cuda.synchronize()
    reps = max(1, steps // G)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(e) / (reps * G) * 1e3
    print(json.dumps({"case": f"dense_fp16_cublas_fc1_b{b}", "m": m, "n": n, "b": b, "us": round(us, 3),
                      "bytes": 2 * m * n, "GBps": round(2 * m * n / (us * 1e-6) / 1e9, 1),
                      "note": "context only: dense fp16 weight (4.7x the packed q=3 bytes), cuBLAS via torch.matmul"}),
          flush=True)
    del Ws
    torch.cuda.empty_cache()


def quantizers(m, n, q, g):
    """Offline step (NEXT-4): time the GPU quantizers on a dense fp16 layer (eager, events)."""
    dev = torch.device("cuda")
    W = (torch.randn(m, n, device=dev) * 0.02).to(torch.float16)
    for name, fn in (("rtn", lambda: L.lutgemm_quantize_rtn(W, q, g)),
                     ("bcq_greedy", lambda: L.lutgemm_quantize_bcq(W, q, g, 0)),
                     ("bcq_alternating_3", lambda: L.lutgemm_quantize_bcq(W, q, g, 3))):
        fn()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        print(json.dumps({"case": f"quantize_{name}", "m": m, "n": n, "q": q, "g": g, "b": 0,
                          "ms": round(a.elapsed_time(e), 3),
                          "GBps_fp16_in": round(2 * m * n / (a.elapsed_time(e) * 1e-3) / 1e9, 1)}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="attn,ffn,llama,batched,dense,quant")
    ap.add_argument("--cases", default="", help="comma list of m:n:q:g[:b[:u]] instead of --only")
    ap.add_argument("--steps", type=int, default=400)
    args = ap.parse_args()
    if args.cases:
        for c in args.cases.split(","):
            f = [int(v) for v in c.split(":")]
            m, n, q, g = f[:4]
            b = f[4] if len(f) > 4 else 1
            u = f[5] if len(f) > 5 else 0  # 1: uniform (App. C), 2: uniform compact format
            case(f"{m}x{n}_q{q}_g{g}_b{b}" + ("_c" if u == 2 else ""), m, n, q, g, b=b, uniform=u >= 1,
                 steps=args.steps, compact=u == 2)
        return
    only = set(args.only.split(","))
    if "ffn" in only:
        case("fc1", 49152, 12288, 3, 128, steps=args.steps)
        case("fc2", 12288, 49152, 3, 128, steps=args.steps)
    if "attn" in only:
        for q in (1, 2, 3, 4):
            for g in (32, 64, 128, 12288):
                case(f"attn_q{q}_g{g}", 12288, 12288, q, g, steps=args.steps)
    if "llama" in only:
        case("llama_8192x8192", 8192, 8192, 4, 128, uniform=True, steps=args.steps)
        case("llama_up_22016x8192", 22016, 8192, 4, 128, uniform=True, steps=args.steps)
        case("llama_down_8192x22016", 8192, 22016, 4, 128, uniform=True, steps=args.steps)
        case("llama_8192x8192_compact", 8192, 8192, 4, 128, uniform=True, steps=args.steps, compact=True)
        case("llama_up_22016x8192_compact", 22016, 8192, 4, 128, uniform=True, steps=args.steps, compact=True)
        case("llama_down_8192x22016_compact", 8192, 22016, 4, 128, uniform=True, steps=args.steps, compact=True)
    if "batched" in only:
        for b in (2, 4, 8, 16, 32):
            case(f"fc1_b{b}", 49152, 12288, 3, 128, b=b, steps=max(20, args.steps // (4 * b)))
    if "quant" in only:
        quantizers(49152, 12288, 3, 128)
    if "dense" in only:
        for b in (1, 2, 4, 8, 16, 32):
            dense_fp16(49152, 12288, b)


if __name__ == "__main__":
    main()
