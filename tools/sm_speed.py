"""Per-SM main-loop speed of the fc1 GEMV over several launches: is the CTA
end-time spread a property of the SM (stable) or noise?"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import gen_bcq, gen_x  # noqa: E402

m, n, q, g = 49152, 12288, 3, 128
d = gen_bcq(5, m, n, q, g)
ws_ = [L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(), torch.from_numpy(d["alpha"]).cuda(),
                          None, n, g) for _ in range(2)]
x = torch.from_numpy(gen_x(1, 1, n)[0]).cuda()
y = torch.empty(m, dtype=torch.float16, device="cuda")
wsb = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
for i in range(4):
    L.lutgemm_gemv(ws_[i % 2], x, y, wsb)
torch.cuda.synchronize()
dur = {}
for r in range(12):
    L.lutgemm_trace_enable(True)
    L.lutgemm_gemv(ws_[r % 2], x, y, wsb)
    torch.cuda.synchronize()
    t = L.lutgemm_trace_read(1024).astype(np.int64)
    t = np.concatenate([t[:512][t[:512, 0] > 0], t[512:][t[512:, 0] > 0]])
    for row in t:
        sm = int(row[7] & 0xFFFFFFFF)
        dur.setdefault(sm, []).append((row[4] - row[2]) / 1e3)  # LUT built -> all warps done
L.lutgemm_trace_enable(False)
sms = sorted(dur)
mean = np.array([np.mean(dur[s]) for s in sms])
std = np.array([np.std(dur[s]) for s in sms])
print(f"SMs {len(sms)}; main-loop us: mean of means {mean.mean():.2f}, spread of means {mean.min():.2f}..{mean.max():.2f}, "
      f"mean within-SM std {std.mean():.2f}")
order = np.argsort(mean)
print("fastest SMs:", [(sms[i], round(mean[i], 2)) for i in order[:8]])
print("slowest SMs:", [(sms[i], round(mean[i], 2)) for i in order[-8:]])
# correlation between launches (first half vs second half)
a = np.array([np.mean(dur[s][:6]) for s in sms])
b = np.array([np.mean(dur[s][6:]) for s in sms])
print("correlation of per-SM means between launch halves:", round(float(np.corrcoef(a, b)[0, 1]), 3))
