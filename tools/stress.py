"""Randomised GPU parity stress over the whole supported space (shapes, q, g kinds,
b 1..32, offset / compact uniform, fp32 output, reducer counts) against the fp64
oracle.  python tools/stress.py [N] [seed]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2206_09557_b200 as L  # noqa: E402
from tests._helpers import parity  # noqa: E402
from workloads import gen_bcq, gen_uniform, gen_x  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main(N=300, seed=1):
    rng = np.random.default_rng(seed)
    worst = (0.0, None)
    done = 0
    while done < N:
        q = int(rng.integers(1, 9))
        n = 32 * int(rng.integers(1, 400))
        kind = rng.integers(0, 3)
        g = int(2 ** rng.integers(5, 11)) if kind == 0 else (1024 * int(rng.integers(1, 5)) if kind == 1 else n)
        if n % g:
            continue
        m = int(rng.integers(1, 6000))
        b = int(rng.choice([1, 1, 1, 2, 2, 3, 4, 4, 5, 8, 16, 31, 32]))
        fmt = int(rng.integers(0, 3))
        f32 = bool(rng.integers(0, 2))
        red = str(int(rng.choice([0, 1, 2, 64])))
        os.environ["LUTGEMM_GEMV_REDUCERS"] = red
        X = gen_x(done, b, n)
        if fmt == 2:
            u = gen_uniform(done, m, n, q, g)
            w = L.lutgemm_pack_uniform(dev(u["codes"]), dev(u["scale"]), dev(u["zero"]), q, g, compact=True)
            planes, alpha, z = O.uniform_to_bcq(u["codes"], u["scale"], u["zero"], q)
            ref = O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(z), X, n, g)
        else:
            d = gen_bcq(done, m, n, q, g, offset=fmt == 1)
            w = L.lutgemm_pack_bcq(dev(d["planes"].view(np.int32)), dev(d["alpha"]),
                                   None if d["offset"] is None else dev(d["offset"]), n, g)
            ref = O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g)
        Xd = dev(X)
        if b == 1 and not f32:
            y = L.lutgemm_gemv(w, Xd[0])[None]
        else:
            y = L.lutgemm_gemm_batched(w, Xd, f32=f32)
        torch.cuda.synchronize()
        y = y.float().cpu().numpy().astype(np.float64)
        pr = parity(y.ravel(), ref.ravel())
        ok = pr["rel_l2"] <= 2e-3 and pr["max_rel"] <= 1e-2
        cfg = (m, n, q, g, b, fmt, f32, red)
        if pr["rel_l2"] > worst[0]:
            worst = (pr["rel_l2"], cfg)
        if not ok:
            print("FAIL", cfg, pr, flush=True)
        done += 1
    print(f"stress: {N} random configs, worst rel-L2 {worst[0]:.2e} at {worst[1]}", flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:3]))
