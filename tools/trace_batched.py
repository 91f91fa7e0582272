"""Per-CTA timeline of sub-slices 2 and 3 of one batched LUT-GEMM launch:
[0] sub-slice start, [1] x staged, [2] LUT built (+ next x issued), [3] warp 0's lookups done."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import gen_bcq, gen_x  # noqa: E402

m, n, q, g, b = 49152, 12288, 3, 128, int(sys.argv[1]) if len(sys.argv) > 1 else 8
d = gen_bcq(3, m, n, q, g)
w = L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(), torch.from_numpy(d["alpha"]).cuda(), None, n, g)
X = torch.from_numpy(gen_x(3, b, n)).cuda()
Y = torch.empty((b, m), dtype=torch.float16, device="cuda")
ws = L.make_workspace(L.lutgemm_workspace_bytes(m, n, b), "cuda")
for _ in range(3):
    L.lutgemm_gemm_batched(w, X, Y, ws)
L.lutgemm_trace_enable(True)
L.lutgemm_gemm_batched(w, X, Y, ws)
torch.cuda.synchronize()
t = L.lutgemm_trace_read(148).astype(np.int64)
for sub in range(2):
    c = t[:, 4 * sub:4 * sub + 4]
    d0 = (c[:, 1] - c[:, 0]) / 1e3
    d1 = (c[:, 2] - c[:, 1]) / 1e3
    d2 = (c[:, 3] - c[:, 2]) / 1e3
    nxt = (t[:, 4] - c[:, 3]) / 1e3 if sub == 0 else None
    print(f"sub-slice {sub + 2}: wait x {np.median(d0):.2f} us, build {np.median(d1):.2f} us, lookups(w0) {np.median(d2):.2f} us"
          + (f", barrier->next start {np.median(nxt):.2f} us" if nxt is not None else ""))
L.lutgemm_trace_enable(False)
