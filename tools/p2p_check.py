"""Fused GEMV + rows all-gather over peer memory (lutgemm_p2p_*), checked against
the plain GEMV of the full (unsharded) layer: every rank's gathered output must be
bitwise equal to the 1-GPU rows (same fixed-order reduction per row).

--mode cols checks the column split (lutgemm_p2p_gemv_allreduce): each rank owns
n/P columns and x's matching slice; every rank's y must be bitwise equal across
ranks and within rel-L2 2e-3 of the 1-GPU GEMV (the fp32 partials are summed in
rank order, a different association than the 1-GPU slice order).

    torchrun --nproc-per-node P tools/p2p_check.py [--same-device] [--rounds 5] [--mode rows|cols]

--same-device puts every rank on cuda:0 (CUDA IPC works between processes on one
GPU; the handles travel over gloo) -- the single-GPU validation of the multi-rank
protocol.  Exits non-zero on a mismatch.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2206_09557_b200 as L  # noqa: E402
from workloads import gen_bcq, gen_x  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--same-device", action="store_true")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--rows", type=int, default=8192)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--timing", action="store_true")
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
    ms = m // world
    d = gen_bcq(11, m, n, q, g)
    if a.mode == "cols":
        return cols(a, rank, world, dev, d, m, n, q, g)
    planes = torch.from_numpy(d["planes"].view(np.int32)).to(dev)
    alpha = torch.from_numpy(d["alpha"]).to(dev)
    full = L.lutgemm_pack_bcq(planes, alpha, None, n, g)
    shard = L.lutgemm_pack_bcq(planes[:, rank * ms:(rank + 1) * ms].contiguous(),
                               alpha[rank * ms:(rank + 1) * ms].contiguous(), None, n, g)
    grp = L.P2PGroup(rank, world, m)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(ms, n, 1), dev)
    wsf = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), dev)
    ok = True
    for r in range(a.rounds):
        x = torch.from_numpy(gen_x(100 + r, 1, n)[0]).to(dev)
        ref = L.lutgemm_gemv(full, x, None, wsf)
        y = torch.empty(m, dtype=torch.float16, device=dev)
        grp.gemv_allgather(shard, x, ws, y)
        torch.cuda.synchronize()
        same = torch.equal(y.view(torch.int16), ref.view(torch.int16))
        ok &= bool(same)
        print(f"rank {rank} round {r}: gathered == 1-GPU rows bitwise: {same}", flush=True)
    if a.timing:  # fused call (GEMV + P2P all-gather + wait) vs the plain shard GEMV, events, eager
        x = torch.from_numpy(gen_x(7, 1, n)[0]).to(dev)
        yl = torch.empty(ms, dtype=torch.float16, device=dev)
        fns = [(lambda: grp.gemv_allgather(shard, x, ws), "fused gemv+allgather (P2P epilogue)"),
               (lambda: L.lutgemm_gemv(shard, x, yl, ws), "shard gemv only")]
        if world == 1:  # the NCCL baseline at world 1: GEMV + ncclAllGather (lutgemm_tp_linear)
            dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29599", world_size=1, rank=0,
                                    device_id=dev)
            comm = L.TPComm(0, 1, device=dev)
            tws = L.make_workspace(comm.workspace_bytes(L.TP_ROWS_ALLGATHER, ms, n, 1), dev)
            yg = torch.empty(m, dtype=torch.float16, device=dev)
            fns.append((lambda: comm.linear(L.TP_ROWS_ALLGATHER, shard, x, yg, tws), "gemv + ncclAllGather"))
        for fn, name in fns:
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(200):
                fn()
            e1.record()
            torch.cuda.synchronize()
            print(f"rank {rank} {name}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us/call", flush=True)
    if world > 1:
        dist.barrier()
    grp.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


def cols(a, rank, world, dev, d, m, n, q, g):
    ns = n // world
    planes = torch.from_numpy(d["planes"].view(np.int32)).to(dev)
    alpha = torch.from_numpy(d["alpha"]).to(dev)
    full = L.lutgemm_pack_bcq(planes, alpha, None, n, g)
    shard = L.lutgemm_pack_bcq(planes[:, :, rank * ns // 32:(rank + 1) * ns // 32].contiguous(),
                               alpha[:, rank * ns // g:(rank + 1) * ns // g].contiguous(), None, ns, g)
    grp = L.P2PGroup(rank, world, m, out_bytes=4 * world * m)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(m, ns, 1), dev)
    wsf = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), dev)
    ok = True
    for r in range(a.rounds):
        x = torch.from_numpy(gen_x(100 + r, 1, n)[0]).to(dev)
        ref = L.lutgemm_gemv(full, x, None, wsf).float()
        y = torch.empty(m, dtype=torch.float16, device=dev)
        grp.gemv_allreduce(shard, x[rank * ns:(rank + 1) * ns].contiguous(), ws, y)
        torch.cuda.synchronize()
        rel = float((y.float() - ref).norm() / ref.norm())
        same = True
        if world > 1:
            ys = [torch.empty(m, dtype=torch.int32) for _ in range(world)]  # gloo: no int16
            dist.all_gather(ys, y.view(torch.int16).cpu().int())
            same = all(torch.equal(t, ys[0]) for t in ys)
        good = rel <= 2e-3 and same
        ok &= good
        print(f"rank {rank} round {r}: allreduce rel-L2 {rel:.2e}, equal across ranks {same}: "
              f"{'PASS' if good else 'FAIL'}", flush=True)
    if a.timing:  # fused call (GEMV + fp32 partial exchange + wait + P-way sum) vs the plain shard GEMV
        xl = torch.from_numpy(gen_x(7, 1, n)[0]).to(dev)[rank * ns:(rank + 1) * ns].contiguous()
        y = torch.empty(m, dtype=torch.float16, device=dev)
        for fn, name in [(lambda: grp.gemv_allreduce(shard, xl, ws, y), "fused gemv+allreduce (P2P epilogue)"),
                         (lambda: L.lutgemm_gemv(shard, xl, y, ws), "shard gemv only")]:
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(200):
                fn()
            e1.record()
            torch.cuda.synchronize()
            print(f"rank {rank} {name}: {e0.elapsed_time(e1) / 200 * 1e3:.2f} us/call", flush=True)
    if world > 1:
        dist.barrier()
    grp.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
