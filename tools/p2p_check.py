"""Fused tensor-parallel GEMV exchange over peer memory (lutgemm_p2p_*), checked
against the fp64 oracle.

    torchrun --nproc-per-node P tools/p2p_check.py [--same-device] [--rounds R] [--mode rows|cols]
                                                   [--graph] [--timing]

rows: rank r owns rows [r m/P, (r+1) m/P) of an m x n layer and the full x; every rank's gathered
      y must match the oracle (north_star tolerances) and be bitwise equal to the 1-GPU GEMV of
      the unsharded layer (each row keeps its fixed-order reduction).
cols: rank r owns columns [r n/P, (r+1) n/P) and x's slice; every rank's y must match the oracle
      and be bitwise equal across ranks (the P partials are summed in rank order on the owner).

The R rounds are issued BACK TO BACK without a host synchronisation (distinct x and y per round),
so the double-buffered flow control runs under real overlap; with --graph they are captured in
one CUDA graph that is replayed twice (the round counter lives on the device).  --same-device
puts every rank on cuda:0 (CUDA IPC works between processes on one GPU; records travel over
gloo): the single-GPU validation of the multi-rank protocol.  Exits non-zero on a mismatch.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_2206_09557_b200 as L  # noqa: E402
from tests._helpers import parity  # noqa: E402
from workloads import gen_bcq, gen_x  # noqa: E402


def timed(fn, iters=200):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--same-device", action="store_true")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--timing", action="store_true")
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--no-oracle", action="store_true", help="skip the oracle (large timing runs)")
    ap.add_argument("--mode", choices=["rows", "cols"], default="rows")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", 0 if a.same_device else local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("gloo")
    m, n, q, g = a.rows, a.cols, 3, 128
    d = gen_bcq(11, m, n, q, g)
    planes = torch.from_numpy(d["planes"].view(np.int32)).to(dev)
    alpha = torch.from_numpy(d["alpha"]).to(dev)
    full = L.lutgemm_pack_bcq(planes, alpha, None, n, g)
    wsf = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), dev)
    if a.mode == "rows":
        ms = m // world
        shard = L.lutgemm_pack_bcq(planes[:, rank * ms:(rank + 1) * ms].contiguous(),
                                   alpha[rank * ms:(rank + 1) * ms].contiguous(), None, n, g)
        grp = L.P2PGroup(rank, world, rows_out=m)
        ws = L.make_workspace(L.lutgemm_workspace_bytes(ms, n, 1), dev)
        xin = lambda x: x  # noqa: E731
        call = lambda x, y: grp.gemv_allgather(shard, x, ws, y)  # noqa: E731
    else:
        ns = n // world
        shard = L.lutgemm_pack_bcq(planes[:, :, rank * ns // 32:(rank + 1) * ns // 32].contiguous(),
                                   alpha[:, rank * ns // g:(rank + 1) * ns // g].contiguous(), None, ns, g)
        grp = L.P2PGroup(rank, world, cols_m=m)
        ws = L.make_workspace(L.lutgemm_workspace_bytes(m, ns, 1), dev)
        xin = lambda x: x[rank * ns:(rank + 1) * ns].contiguous()  # noqa: E731
        call = lambda x, y: grp.gemv_allreduce(shard, x, ws, y)  # noqa: E731
    del planes, alpha

    R = a.rounds
    xs_host = [gen_x(100 + r, 1, n) for r in range(R)]
    xs = [xin(torch.from_numpy(x[0]).to(dev)) for x in xs_host]
    ys = [torch.full((m,), float("nan"), dtype=torch.float16, device=dev) for _ in range(R)]
    refs = [L.lutgemm_gemv(full, torch.from_numpy(x[0]).to(dev), None, wsf) for x in xs_host]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    def issue():
        for r in range(R):
            call(xs[r], ys[r])

    if a.graph:
        issue()  # eager warm-up rounds (also exercise the protocol once more)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(graph, stream=cap):
            issue()
        for y in ys:
            y.fill_(float("nan"))
        graph.replay()
        graph.replay()
    else:
        issue()  # back to back, no host synchronisation between rounds
    torch.cuda.synchronize()

    ok = True
    for r in range(R):
        y = ys[r]
        p = None
        if not a.no_oracle:
            p = parity(y.float().cpu().numpy(), O.bcq_gemv(d["planes"], d["alpha"], None, xs_host[r], n, g)[0])
        good = p is None or (p["rel_l2"] <= 2e-3 and p["max_rel"] <= 1e-2)
        if a.mode == "rows":
            same = torch.equal(y.view(torch.int16), refs[r].view(torch.int16))
            what = "bitwise == 1-GPU rows"
        else:
            same = True
            if world > 1:
                yy = [torch.empty(m, dtype=torch.int32) for _ in range(world)]  # gloo: no int16
                dist.all_gather(yy, y.view(torch.int16).cpu().int())
                same = all(torch.equal(t, yy[0]) for t in yy)
            what = "bitwise equal across ranks"
        good = good and bool(same)
        ok &= good
        print(f"rank {rank} {a.mode} round {r}: oracle {p}, {what}: {same}: {'PASS' if good else 'FAIL'}", flush=True)

    if a.timing:  # fused call vs the plain shard GEMV, eager back-to-back calls, CUDA events
        x, y = xs[0], ys[0]
        yl = torch.empty(m, dtype=torch.float16, device=dev)
        print(f"rank {rank} fused {a.mode} exchange: {timed(lambda: call(x, y)):.2f} us/call", flush=True)
        print(f"rank {rank} shard gemv only: {timed(lambda: L.lutgemm_gemv(shard, x, yl, ws)):.2f} us/call", flush=True)
    if world > 1:
        dist.barrier()
    grp.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
