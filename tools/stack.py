"""BASELINE config 5: the full OPT-175B decoder linear stack (96 layers x
{QKV 36864x12288, out 12288x12288, fc1 49152x12288, fc2 12288x49152}, q=3,
g=128), one token (b=1), per-token latency on 1 GPU or tensor-parallel.

    python tools/stack.py [--layers 96] [--tokens 20] [--check] [--tp-impl nccl|p2p]
    torchrun --nproc-per-node P tools/stack.py [--tp-impl p2p [--same-device]] ...

Tensor parallelism (Megatron pairing): QKV and fc1 are split by
rows (no communication), out-proj and fc2 by columns -- each rank's input is
its own QKV / fc1 output slice -- followed by an fp32 all-reduce of y
(lutgemm_tp_linear COLS_ALLREDUCE with NCCL, or --tp-impl p2p: the reduce-scatter + all-gather
fused into the GEMV epilogue over peer memory, lutgemm_p2p_gemv_allreduce): 2 all-reduces per layer.
--same-device (p2p only) runs every rank on cuda:0 through CUDA IPC: the single-GPU validation of the
multi-rank path (NCCL refuses two ranks on one GPU).  Attention, LN
and embeddings are omitted (the path is the linears): out-proj reads the first
12288/P outputs of QKV.  Weights are seeded synthetic BCQ (device RNG), 73.4 GB
at P=1.  One token = one CUDA graph of 384 LUT-GEMMs (+ 192 all-reduces).

--shard-tp N (world 1): rank 0's shards of TP N run without any exchange -- the per-GPU compute of
TP-N per-token latency, the part one GPU can measure (the exchange adds 2 collectives per layer).

--tp-scheme allgather: the contrast variant of SURVEY 8(e) -- every linear split by rows and its y
all-gathered (4 collectives per layer, 384 per token) instead of the Megatron pairing.

--check: for layers 0 and L-1 each linear is also run on a seeded x and 64
sampled rows are compared with the fp64 oracle (its inputs are the seeded
canonical weights copied to the host before packing, never a CUDA output);
the column-split linears through the actual TP exchange (the oracle partials of
every rank's shard summed across ranks).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2206_09557_b200 as L  # noqa: E402

H = 12288
LINEARS = [("qkv", 3 * H, H, "rows"), ("out", H, H, "cols"), ("fc1", 4 * H, H, "rows"), ("fc2", H, 4 * H, "cols")]
Q, G = 3, 128


def gen_canonical(seed: int, m: int, n: int, dev):
    """Device-generated canonical BCQ (same distributions as workloads.gen_bcq)."""
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    planes = torch.randint(0, 256, (Q, m, n // 32 * 4), dtype=torch.uint8, device=dev, generator=gen)
    planes = planes.view(torch.int32)
    u = torch.rand((m, n // G, Q), device=dev, generator=gen) * 0.5 + 0.75
    alpha = (0.87 * (2.0 ** -torch.arange(Q, device=dev)) * u / math.sqrt(n)).to(torch.float16)
    return planes.contiguous(), alpha.contiguous()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=96)
    ap.add_argument("--tokens", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--tp-impl", default="nccl", choices=["nccl", "p2p"])
    ap.add_argument("--same-device", action="store_true")
    ap.add_argument("--shard-tp", type=int, default=0,
                    help="world 1 only: run rank 0's shards of TP N (1/2/4/8) without the exchange")
    ap.add_argument("--tp-scheme", default="megatron", choices=["megatron", "allgather"],
                    help="megatron: QKV / fc1 by rows, out / fc2 by columns + all-reduce (2 collectives per "
                         "layer); allgather: every linear by rows + all-gather of y (4 per layer, the contrast "
                         "variant of SURVEY 8(e))")
    ap.add_argument("--arena", action="store_true",
                    help="all packed weights in one device allocation (2 MB aligned views)")
    ap.add_argument("--graph-layers", type=int, default=0,
                    help="layers per CUDA graph (default: the whole token in one graph)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # shard size: the TP degree (or, at world 1, --shard-tp N: rank 0's shards of TP N without the
    # exchange -- the per-GPU compute part of TP-N latency, measurable on one GPU)
    sw = world
    if args.shard_tp:
        if world > 1:
            raise SystemExit("--shard-tp is a world-1 option")
        sw = args.shard_tp
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", 0 if args.same_device else local)
    torch.cuda.set_device(dev)
    comm = p2p = None
    if world > 1:
        import torch.distributed as dist
        if args.tp_impl == "nccl":
            dist.init_process_group("nccl", device_id=dev)
            comm = L.TPComm(rank, world, device=dev)
        else:
            dist.init_process_group("gloo")
    ag = args.tp_scheme == "allgather"
    linears = [(nm, m, n, "rows" if ag else sp) for nm, m, n, sp in LINEARS]
    if args.tp_impl == "p2p":
        p2p = L.P2PGroup(rank, world, rows_out=4 * H if ag else 0, cols_m=0 if ag else H)

    t0 = time.time()
    arena, aoff = None, 0
    if args.arena:
        A2 = 2 << 20
        sizes = [(L.lutgemm_packed_bytes(m // sw, n, Q, G, False) if s == "rows" else
                  L.lutgemm_packed_bytes(m, n // sw, Q, G, False)) for _, m, n, s in linears]
        arena = torch.empty(args.layers * sum((z + A2 - 1) // A2 * A2 for z in sizes) + A2, dtype=torch.uint8,
                            device=dev)
        aoff = (-arena.data_ptr()) % A2
    weights = []  # per layer: dict name -> PackedBCQ
    check_rows = {}
    rng = np.random.default_rng(0)
    for layer in range(args.layers):
        lw = {}
        for li, (name, m, n, split) in enumerate(linears):
            ms, ns = (m // sw, n) if split == "rows" else (m, n // sw)
            seed = 1_000_003 * layer + 1009 * li + rank
            planes, alpha = gen_canonical(seed, ms, ns, dev)
            if args.check and layer in (0, args.layers - 1):
                rows = np.sort(rng.choice(ms, size=64, replace=False))
                idx = torch.from_numpy(rows).to(dev)
                check_rows[(layer, name)] = (rows, planes[:, idx].cpu().numpy().view(np.uint32),
                                             alpha[idx].cpu().numpy(), ms, ns)
            out = None
            if arena is not None:
                nb = L.lutgemm_packed_bytes(ms, ns, Q, G, False)
                out = arena[aoff:aoff + nb]
                aoff += (nb + (2 << 20) - 1) // (2 << 20) * (2 << 20)
            lw[name] = L.lutgemm_pack_bcq(planes, alpha, None, ns, G, out=out)
            del planes, alpha
        weights.append(lw)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    mem_gb = torch.cuda.memory_allocated(dev) / 1e9

    # activations (each rank: full x; local QKV/fc1 outputs; replicated out/fc2 outputs)
    gx = torch.Generator(device=dev)
    gx.manual_seed(2206)
    x0 = torch.randn(H, device=dev, generator=gx).to(torch.float16)  # seeded: x_sha is reproducible
    x = x0.clone()
    # (allgather: every output is gathered to its full length)
    qkv_o = torch.empty(3 * H if ag else 3 * H // sw, dtype=torch.float16, device=dev)
    out_o = torch.empty(H, dtype=torch.float16, device=dev)
    fc1_o = torch.empty(4 * H if ag else 4 * H // sw, dtype=torch.float16, device=dev)
    ws_bytes = max(L.lutgemm_workspace_bytes(m // sw if s == "rows" else m, n if s == "rows" else n // sw, 1)
                   for _, m, n, s in linears)
    ws = L.make_workspace(ws_bytes, dev)
    tws = None
    if comm is not None:
        if ag:
            tws = L.make_workspace(max(comm.workspace_bytes(L.TP_ROWS_ALLGATHER, m // sw, n, 1)
                                       for _, m, n, _s in linears), dev)
        else:
            tws = L.make_workspace(max(comm.workspace_bytes(L.TP_COLS_ALLREDUCE, H, H // sw, 1),
                                       comm.workspace_bytes(L.TP_COLS_ALLREDUCE, H, 4 * H // sw, 1)), dev)

    def cols(w, xin, y):
        if p2p is not None:
            p2p.gemv_allreduce(w, xin, ws, y)
        elif comm is None:
            L.lutgemm_gemv(w, xin, y, ws)
        else:
            comm.linear(L.TP_COLS_ALLREDUCE, w, xin, y, tws)

    def rows_ag(w, xin, y):  # row shard + all-gather of y (the allgather scheme)
        if p2p is not None:
            p2p.gemv_allgather(w, xin, ws, y)
        elif comm is None:
            L.lutgemm_gemv(w, xin, y, ws)
        else:
            comm.linear(L.TP_ROWS_ALLGATHER, w, xin, y, tws)

    def token(l0=0, l1=None):
        if l0 == 0:
            x.copy_(x0)  # every token starts from the same input (device-to-device copy)
        for lw in weights[l0:l1]:
            if ag:
                rows_ag(lw["qkv"], x, qkv_o)
                rows_ag(lw["out"], qkv_o[:H], out_o)
                rows_ag(lw["fc1"], out_o, fc1_o)
                rows_ag(lw["fc2"], fc1_o, x)
                continue
            L.lutgemm_gemv(lw["qkv"], x, qkv_o, ws)
            cols(lw["out"], qkv_o[:H // sw], out_o)
            L.lutgemm_gemv(lw["fc1"], out_o, fc1_o, ws)
            cols(lw["fc2"], fc1_o, x)

    token()
    torch.cuda.synchronize()
    gl = args.graph_layers if args.graph_layers > 0 else args.layers
    graphs = []
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    for l0 in range(0, args.layers, gl):
        graphs.append(torch.cuda.CUDAGraph())
        with torch.cuda.graph(graphs[-1], stream=cap):
            token(l0, l0 + gl)

    class _Token:  # one token = the graphs in order
        @staticmethod
        def replay():
            for gr in graphs:
                gr.replay()
    graph = _Token
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.tokens):
        graph.replay()
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e) / args.tokens
    if world > 1:
        t = torch.tensor([ms], device=dev if comm is not None else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t[0])
    finite = bool(torch.isfinite(x.float()).all())
    import hashlib
    x_sha = hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()[:16]  # the token's output (bitwise check)

    # per-linear breakdown on this rank (eager, events around each call of one layer)
    per = {}
    for name in ("qkv", "out", "fc1", "fc2"):
        lw = weights[args.layers // 2]
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        xin, y = {"qkv": (x, qkv_o), "out": (qkv_o[:H] if ag else qkv_o[:H // sw], out_o), "fc1": (out_o, fc1_o),
                  "fc2": (fc1_o, x)}[name]

        def one():
            if ag:
                rows_ag(lw[name], xin, y)
            elif name in ("qkv", "fc1"):
                L.lutgemm_gemv(lw[name], xin, y, ws)
            else:
                cols(lw[name], xin, y)
        for _ in range(3):
            one()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(20):
            one()
        ev1.record()
        torch.cuda.synchronize()
        per[name] = round(ev0.elapsed_time(ev1) / 20 * 1e3, 2)

    # parity on layers 0 and L-1 with a seeded x (oracle inputs never come from the GPU)
    parity = {}
    if args.check:
        import oracle as O
        for (layer, name), (rows, planes_rows, alpha_rows, ms_, ns_) in sorted(check_rows.items()):
            xs = np.random.default_rng(layer * 7 + len(name)).standard_normal(ns_).astype(np.float16)
            y = torch.empty(ms_, dtype=torch.float16, device=dev)
            L.lutgemm_gemv(weights[layer][name], torch.from_numpy(xs).to(dev), y, ws)
            torch.cuda.synchronize()
            got = y.float().cpu().numpy()[rows].astype(np.float64)
            ref = O.bcq_gemv(planes_rows, alpha_rows, None, xs[None], ns_, G)[0]
            parity[f"L{layer}.{name}"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
            if ag and (world > 1 or p2p is not None):
                # the gathered output: this rank's rows sit at rank * m_shard of the full vector
                yfull = torch.empty(ms_ * world, dtype=torch.float16, device=dev)
                rows_ag(weights[layer][name], torch.from_numpy(xs).to(dev), yfull)
                torch.cuda.synchronize()
                got = yfull.float().cpu().numpy()[rank * ms_ + rows].astype(np.float64)
                parity[f"L{layer}.{name}.tp"] = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
            elif name in ("out", "fc2") and (world > 1 or p2p is not None):
                # the TP output of the column split: sum over ranks of each shard's oracle partial
                xf = np.random.default_rng(layer * 7 + len(name) + 1).standard_normal(ns_ * world).astype(np.float16)
                xl = xf[rank * ns_:(rank + 1) * ns_]
                cols(weights[layer][name], torch.from_numpy(xl).to(dev), y)
                torch.cuda.synchronize()
                part = O.bcq_gemv(planes_rows, alpha_rows, None, xl[None], ns_, G)[0]
                if world > 1:
                    t = torch.from_numpy(part).to(dev if comm is not None else "cpu")
                    torch.distributed.all_reduce(t)
                    part = t.cpu().numpy()
                got = y.float().cpu().numpy()[rows].astype(np.float64)
                parity[f"L{layer}.{name}.tp"] = float(np.linalg.norm(got - part) / np.linalg.norm(part))

    bytes_token = sum(((m // sw) * n if s == "rows" else m * (n // sw)) * (Q / 8 + 2 * Q / G)
                      for _, m, n, s in linears) * args.layers
    if rank == 0:
        print(json.dumps({
            "config": "OPT-175B decoder linear stack (96 x QKV/out/fc1/fc2), q=3 g=128, b=1",
            "layers": args.layers, "graph_layers": gl, "arena": args.arena, "tp": world,
            "shard_tp": sw if args.shard_tp else None, "tp_impl": args.tp_impl if world > 1 or p2p else None,
            "x_sha": x_sha,
            "ms_per_token": round(ms, 4),
            "GBps_per_gpu": round(bytes_token / (ms * 1e-3) / 1e9, 1),
            "weight_bytes_per_gpu": int(bytes_token), "tp_scheme": args.tp_scheme,
            "allreduces_per_token": 2 * args.layers if world > 1 and not ag else 0,
            "allgathers_per_token": 4 * args.layers if world > 1 and ag else 0,
            "per_linear_us_eager": per, "finite": finite, "build_s": round(build_s, 1),
            "hbm_alloc_gb": round(mem_gb, 1), "parity_rel_l2_sampled": parity,
            "paper_context_ms": "A100 FT e2e per token, 3-bit row-wise: 51.6 (1 GPU), 35.8 (2), 27.2 (4), 24.2 (8) (Table 4 P:L475-478)",
        }), flush=True)
    if p2p is not None:
        p2p.close()
    if comm is not None:
        comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
