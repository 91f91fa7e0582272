"""Does the number of distinct weight buffers a GEMV chain walks change the per-GEMV time?

The sweep chains GEMVs over 2-4 rotating copies (510 MB); the 96-layer stack walks 73 GB of
distinct weights.  This times the same shape in a CUDA-graph chain over k distinct packed copies
(k = 2 ... 32) to separate address-translation / first-touch costs from the kernel itself.

    python tools/tlb_probe.py [--cases 49152:12288,12288:12288] [--copies 2,8,32]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2206_09557_b200 as L  # noqa: E402
from sweep import time_product  # noqa: E402
from workloads import gen_bcq, gen_x  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="49152:12288,12288:12288")
    ap.add_argument("--copies", default="2,8,32")
    ap.add_argument("--steps", type=int, default=400)
    args = ap.parse_args()
    dev = torch.device("cuda")
    for c in args.cases.split(","):
        m, n = (int(v) for v in c.split(":"))
        d = gen_bcq(7, m, n, 3, 128)
        planes = torch.from_numpy(d["planes"].view(np.int32)).to(dev)
        alpha = torch.from_numpy(d["alpha"]).to(dev)
        X = torch.from_numpy(gen_x(7, 1, n)).to(dev)
        for k in (int(v) for v in args.copies.split(",")):
            ws = [L.lutgemm_pack_bcq(planes, alpha, None, n, 128) for _ in range(k)]
            chain, iso = time_product(ws, X, 1, m, n, max(args.steps, k))
            print(json.dumps({"m": m, "n": n, "copies": k, "chain_us": round(chain, 3), "iso_us": round(iso, 3),
                              "distinct_MB": round(k * ws[0].nbytes() / 1e6, 1)}),
                  flush=True)
            del ws
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
