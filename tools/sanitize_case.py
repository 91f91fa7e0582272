"""Small products through every kernel path, for compute-sanitizer runs:
GEMV (fused reductions: one reducer and many), batched V=2 / V=4, compact
uniform format, n and m tails, fp32 output, every layout group class (straddling
groups, per-chunk scales, partial last lane).  Checks results against the oracle."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import gen_bcq, gen_uniform, gen_x  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(y, ref, what):
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert rel < 2e-3, (what, rel)
    print(f"ok {what} rel-L2 {rel:.2e}", flush=True)


def main():
    for (m, n, q, g, b, off) in [(512, 512, 3, 128, 1, False), (777, 5152, 4, 32, 1, True), (6000, 4096, 3, 128, 1, False), (2049, 2048, 2, 64, 1, False),
                                 (333, 1536, 3, 128, 2, True), (130, 5152, 3, 32, 5, False), (64, 2048, 6, 2048, 32, True),
                                 # SURVEY 8(b) shapes: groups straddling slices, chunk groups (g % 32 != 0, the
                                 # generic-q kernels' per-chunk scales), n % 32 != 0; a 15-slice fused grid
                                 (300, 4800, 3, 96, 1, True), (257, 4104, 3, 24, 1, True), (129, 4104, 3, 24, 3, True),
                                 (200, 2040, 2, 40, 6, False), (900, 4104, 3, 4104, 2, True), (64, 15360, 3, 128, 1, False)]:
        d = gen_bcq(m + n + b, m, n, q, g, offset=off)
        X = gen_x(m + b, b, n)
        w = L.lutgemm_pack_bcq(dev(d["planes"].view(np.int32)), dev(d["alpha"]),
                               None if d["offset"] is None else dev(d["offset"]), n, g)
        Xd = dev(X)
        y = (L.lutgemm_gemv(w, Xd[0])[None] if b == 1 else L.lutgemm_gemm_batched(w, Xd)).float().cpu().numpy()
        check(y.astype(np.float64), O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g), (m, n, q, g, b))
        yf = L.lutgemm_gemm_batched(w, Xd, f32=True).cpu().numpy()
        check(yf.astype(np.float64), O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g), ("f32", m, n, b))
    for b in (1, 4):
        m, n, q, g = 300, 3072, 4, 128
        u = gen_uniform(7 + b, m, n, q, g)
        X = gen_x(3, b, n)
        w = L.lutgemm_pack_uniform(dev(u["codes"]), dev(u["scale"]), dev(u["zero"]), q, g, compact=True)
        y = (L.lutgemm_gemv(w, dev(X)[0])[None] if b == 1 else L.lutgemm_gemm_batched(w, dev(X))).float().cpu().numpy()
        planes, alpha, z = O.uniform_to_bcq(u["codes"], u["scale"], u["zero"], q)
        check(y.astype(np.float64), O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(z), X, n, g), ("compact", b))
    # quantizers (NEXT-4): RTN and greedy / alternating BCQ, bit-exact vs the oracle
    import oracle.quantize_oracle as Q
    rng = np.random.default_rng(3)
    W = (rng.standard_normal((9, 1024)) * 0.05).astype(np.float16)
    c, sc, z = L.lutgemm_quantize_rtn(dev(W), 3, 128)
    rc, rs, rz = Q.quantize_rtn(W, 3, 128)
    assert np.array_equal(c.cpu().numpy(), rc) and np.array_equal(sc.cpu().numpy(), rs)
    print("ok quantize_rtn", flush=True)
    for iters in (0, 2):
        p, a = L.lutgemm_quantize_bcq(dev(W), 3, 128, iters)
        rp, ra = Q.quantize_bcq_greedy(W, 3, 128) if iters == 0 else Q.quantize_bcq_alternating(W, 3, 128, iters)
        assert np.array_equal(p.cpu().numpy().view(np.uint32), rp) and np.array_equal(a.cpu().numpy(), ra)
        print(f"ok quantize_bcq iters={iters}", flush=True)
    # fused rows all-gather over peer memory (NEXT-1), world 1
    m, n = 6000, 4096
    d = gen_bcq(9, m, n, 3, 128)
    w = L.lutgemm_pack_bcq(dev(d["planes"].view(np.int32)), dev(d["alpha"]), None, n, 128)
    grp = L.P2PGroup(0, 1, rows_out=m)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
    for r in range(3):
        x = dev(gen_x(r, 1, n)[0])
        y = torch.empty(m, dtype=torch.float16, device="cuda")
        grp.gemv_allgather(w, x, ws, y)
        ref = L.lutgemm_gemv(w, x)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16))
    grp.close()
    grp = L.P2PGroup(0, 1, cols_m=m)  # fused column reduce-scatter + all-gather
    for r in range(3):
        x = dev(gen_x(r, 1, n)[0])
        y = torch.empty(m, dtype=torch.float16, device="cuda")
        grp.gemv_allreduce(w, x, ws, y)
        ref = L.lutgemm_gemv(w, x)
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16))
    grp.close()
    print("ok p2p world 1", flush=True)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
