"""Per-CTA timeline of one LUT-GEMM GEMV launch (lutgemm_trace_enable), to see
where the kernel's time goes (start-up, LUT build, streaming, epilogue, tail).

    python tools/trace_gemv.py [config]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import CONFIGS, gen_bcq, gen_x  # noqa: E402


def main(name="fc1", reps=3):
    if name in CONFIGS:
        c = CONFIGS[name]
        m, n, q, g, seed = c["m"], c["n"], c["q"], c["g"], c["seed"]
    else:  # "m,n,q,g"
        m, n, q, g = (int(v) for v in name.split(","))
        seed = 5
    d = gen_bcq(seed, m, n, q, g)
    ws_ = [L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(), torch.from_numpy(d["alpha"]).cuda(),
                              None, n, g) for _ in range(2)]
    x = torch.from_numpy(gen_x(1, 1, n)[0]).cuda()
    y = torch.empty(m, dtype=torch.float16, device="cuda")
    wsb = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
    for i in range(10):
        L.lutgemm_gemv(ws_[i % 2], x, y, wsb)
    L.lutgemm_trace_enable(True)
    for r in range(reps):
        L.lutgemm_trace_enable(True)  # clears nothing: stale CTAs are filtered by a zero start below
        L.lutgemm_gemv(ws_[r % 2], x, y, wsb)
        torch.cuda.synchronize()
        t = L.lutgemm_trace_read(1024).astype(np.int64)
        t = np.concatenate([t[:512][t[:512, 0] > 0], t[512:][t[512:, 0] > 0]])
        nsl = t[:, 7] >> 32
        t[:, 7] &= 0xFFFFFFFF
        t0 = t[:, 0].min()
        rel = (t[:, :7] - t0) / 1000.0
        print(f"--- launch {r}: LUT kernel span {max(rel[:, 6].max(), rel[:, 4].max()):.2f} us (ns timer)")
        names = ["start", "x staged", "LUT built", "w0 slice1 end", "slice1 done", "pdl wait done", "CTA end"]
        for k, nm in enumerate(names):
            col = rel[:, k][t[:, k] > 0]
            if len(col):
                print(f"  {nm:12s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
        end = np.where(t[:, 6] > 0, rel[:, 6], rel[:, 4])
        print("  slices per CTA histogram:", {int(k): int(v) for k, v in zip(*np.unique(nsl, return_counts=True))})
        order = np.argsort(end)
        print("  latest CTAs (cta, sm, end us):", [(int(i), int(t[i, 7]), round(float(end[i]), 2)) for i in order[-6:]])
        print("  earliest CTAs:", [(int(i), int(t[i, 7]), round(float(end[i]), 2)) for i in order[:6]])
    L.lutgemm_trace_enable(False)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["fc1"]))
