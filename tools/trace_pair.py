"""Timeline of two consecutive GEMVs captured in one CUDA graph (PDL-chained):
where the time between the end of one LUT kernel and the streaming of the next goes.

    python tools/trace_pair.py m,n,q,g
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import gen_bcq, gen_x  # noqa: E402

m, n, q, g = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "12288,12288,3,128").split(","))
d = gen_bcq(5, m, n, q, g)
ws_ = [L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(), torch.from_numpy(d["alpha"]).cuda(),
                          None, n, g) for _ in range(2)]
x = torch.from_numpy(gen_x(1, 1, n)[0]).cuda()
y = torch.empty(m, dtype=torch.float16, device="cuda")
wsb = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
for i in range(4):
    L.lutgemm_gemv(ws_[i % 2], x, y, wsb)
torch.cuda.synchronize()
L.lutgemm_trace_enable(True)
graph = torch.cuda.CUDAGraph()
cap = torch.cuda.Stream()
cap.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(graph, stream=cap):
    for i in range(2):
        L.lutgemm_gemv(ws_[i], x, y, wsb)
for _ in range(3):
    graph.replay()
torch.cuda.synchronize()
t = L.lutgemm_trace_read(1024).astype(np.int64)
a, b = t[:512], t[512:]
a, b = a[a[:, 0] > 0], b[b[:, 0] > 0]
t0 = min(a[:, 0].min(), b[:, 0].min())
first, second = (a, b) if a[:, 0].min() < b[:, 0].min() else (b, a)
names = ["start", "x staged", "LUT built", "w0 loop end", "all warps done", "group complete", "reduced+depart"]
for lab, tt in (("GEMV 1", first), ("GEMV 2", second)):
    rel = (tt[:, :7] - t0) / 1e3
    print(lab)
    for k, nm in enumerate(names):
        col = rel[:, k][tt[:, k] > 0]
        if len(col):
            print(f"  {nm:14s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
L.lutgemm_trace_enable(False)
