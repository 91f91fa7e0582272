"""Where does the GEMV's fixed cost go?  Per-CTA timelines (lutgemm_trace_enable, %globaltimer)
over many launches: start-up (launch -> x staged -> LUT built), main-loop duration per SM, the
end-time spread across CTAs, and the group reduction.  Asks whether slow SMs are the same SMs
from launch to launch (a per-SM property a static rebalance could exploit) or random.

    python tools/trace_spread.py [m,n,q,g ...]   (default: fc1 and 12288^2)

Prints one JSON line per shape.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import gen_bcq, gen_x  # noqa: E402


def one(m, n, q, g, reps=24, chain=False):
    d = gen_bcq(5, m, n, q, g)
    ws_ = [L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(),
                              torch.from_numpy(d["alpha"]).cuda(), None, n, g) for _ in range(4)]
    x = torch.from_numpy(gen_x(1, 1, n)[0]).cuda()
    y = torch.empty(m, dtype=torch.float16, device="cuda")
    wsb = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
    for i in range(8):
        L.lutgemm_gemv(ws_[i % 4], x, y, wsb)
    torch.cuda.synchronize()
    runs = []
    for r in range(reps):
        L.lutgemm_trace_enable(True)
        if chain:  # the traced launch follows another GEMV through PDL (the decoder situation)
            L.lutgemm_trace_enable(False)
            L.lutgemm_gemv(ws_[(r + 1) % 4], x, y, wsb)
            L.lutgemm_trace_enable(True)
        L.lutgemm_gemv(ws_[r % 4], x, y, wsb)
        torch.cuda.synchronize()
        t = L.lutgemm_trace_read(1024).astype(np.int64)
        t = np.concatenate([t[:512][t[:512, 0] > 0], t[512:][t[512:, 0] > 0]])
        t[:, 7] &= 0xFFFFFFFF
        runs.append(t)
    L.lutgemm_trace_enable(False)
    # per launch: times relative to the earliest CTA start
    stats = {k: [] for k in ("start_skew", "start_to_pdl", "pdl_to_x", "lut_build", "loop_med", "loop_spread",
                             "end_spread", "group_wait", "reduce", "span")}
    per_sm = {}
    for t in runs:
        t0 = t[:, 0].min()
        rel = (t[:, :7] - t0) / 1e3
        loop = rel[:, 4] - rel[:, 2]
        stats["start_skew"].append(float(np.median(rel[:, 0])))
        stats["start_to_pdl"].append(float(np.median(rel[:, 3] - rel[:, 0])))
        stats["pdl_to_x"].append(float(np.median(rel[:, 1] - rel[:, 3])))
        stats["lut_build"].append(float(np.median(rel[:, 2] - rel[:, 1])))
        stats["loop_med"].append(float(np.median(loop)))
        stats["loop_spread"].append(float(loop.max() - loop.min()))
        stats["end_spread"].append(float(rel[:, 4].max() - np.median(rel[:, 4])))
        red = t[:, 6] > 0
        if red.any():
            stats["group_wait"].append(float(np.median(rel[red, 5] - rel[red, 4])))
            stats["reduce"].append(float(np.median(rel[red, 6] - rel[red, 5])))
            stats["span"].append(float(rel[red, 6].max()))
        for sm, lp in zip(t[:, 7], loop):
            per_sm.setdefault(int(sm), []).append(float(lp))
    # is a slow SM slow every time?  split the launches in halves, rank-correlate the per-SM means
    sms = sorted(k for k, v in per_sm.items() if len(v) >= 4)
    a = np.array([np.mean(per_sm[s][: len(per_sm[s]) // 2]) for s in sms])
    b = np.array([np.mean(per_sm[s][len(per_sm[s]) // 2:]) for s in sms])
    ra, rb = np.argsort(np.argsort(a)), np.argsort(np.argsort(b))
    rho = float(np.corrcoef(ra, rb)[0, 1]) if len(sms) > 2 else None
    mean_sm = np.array([np.mean(per_sm[s]) for s in sms])
    slow = [int(sms[i]) for i in np.argsort(mean_sm)[-8:]]
    out = {"shape": [m, n, q, g], "chain": chain, "reps": reps, "ctas": int(len(runs[0])),
           "median_us": {k: round(float(np.median(v)), 3) for k, v in stats.items() if v},
           "per_sm_loop_us": {"min": round(float(mean_sm.min()), 3), "median": round(float(np.median(mean_sm)), 3),
                              "max": round(float(mean_sm.max()), 3)},
           "per_sm_rank_corr_between_halves": rho, "slowest_sms": slow,
           "die_loop_us": {"sm<74": round(float(np.mean([np.mean(per_sm[s]) for s in sms if s < 74])), 3),
                           "sm>=74": round(float(np.mean([np.mean(per_sm[s]) for s in sms if s >= 74])), 3)}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    shapes = sys.argv[1:] or ["49152,12288,3,128", "12288,12288,3,128"]
    for s in shapes:
        m, n, q, g = (int(v) for v in s.split(","))
        one(m, n, q, g, chain=False)
        one(m, n, q, g, chain=True)
