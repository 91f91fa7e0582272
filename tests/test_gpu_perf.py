"""Performance assertions (tier T5): the north-star target -- the q=3,
g=128 GEMV on OPT-175B's FFN layers at >= 70 % of the measured HBM peak
(MEASURED_PEAKS.json) -- and the batched kernel's fraction of the shared-memory
lookup roof.  Timing as bench.py: CUDA graph of consecutive products on rotating
weight copies (> 3x L2), events around the replays."""
import json
import math
import os

import numpy as np
import pytest
import torch

from workloads import gen_bcq, gen_x

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return float(json.load(open(p))["hbm_gbs"]) if os.path.exists(p) else 6650.0


def time_us(m, n, q, g, b, steps=300):
    import paper_2206_09557_b200 as L
    dev = torch.device("cuda")
    d = gen_bcq(5, m, n, q, g)
    planes = torch.from_numpy(d["planes"].view(np.int32)).to(dev)
    alpha = torch.from_numpy(d["alpha"]).to(dev)
    B = m * n * q // 8 + 2 * m * (n // g) * q
    nc = max(2, math.ceil(3 * torch.cuda.get_device_properties(dev).L2_cache_size / B))
    ws = [L.lutgemm_pack_bcq(planes, alpha, None, n, g) for _ in range(nc)]
    X = torch.from_numpy(gen_x(5, b, n)).to(dev)
    Y = torch.empty((b, m), dtype=torch.float16, device=dev)
    wsb = L.make_workspace(L.lutgemm_workspace_bytes(m, n, b), dev)

    def step(i):
        if b == 1:
            L.lutgemm_gemv(ws[i % nc], X[0], Y[0], wsb)
        else:
            L.lutgemm_gemm_batched(ws[i % nc], X, Y, wsb)

    for i in range(4):
        step(i)
    torch.cuda.synchronize()
    G = nc * max(1, 40 // nc)
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=cap):
        for i in range(G):
            step(i)
    graph.replay()
    torch.cuda.synchronize()
    reps = max(1, steps // G)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        graph.replay()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / (reps * G) * 1e3, B + 2 * n * b + 2 * m * b


@pytest.mark.parametrize("m,n,floor", [(49152, 12288, 0.70), (12288, 49152, 0.70)])
def test_ffn_gemv_hbm_fraction(m, n, floor):
    us, B = time_us(m, n, 3, 128, 1)
    frac = B / (us * 1e-6) / 1e9 / peak_gbs()
    print(f"{m}x{n}: {us:.2f} us, {100 * frac:.1f} % of the measured HBM peak")
    assert frac >= floor, f"{us:.2f} us = {100 * frac:.1f} % < {100 * floor:.0f} % of peak"


def test_batched_lds_roof_fraction():
    m, n, q, g, b = 49152, 12288, 3, 128, 8
    us, _ = time_us(m, n, q, g, b, steps=60)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    lds_us = m * q * (n // 8) * b / 32 / sms / 1.965e9 * 1e6  # 128 B/clk/SM of fp32 lookups
    print(f"fc1 b=8: {us:.1f} us, {100 * lds_us / us:.1f} % of the shared-memory roof")
    assert lds_us / us >= 0.5
