#!/usr/bin/env python
"""LUT-GEMM benchmark (BASELINE.json metric: "LUT-GEMM GEMV us and achieved HBM
GB/s (% of B200 peak) at q=3,g=128").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lutgemm|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one pass of the hot path: one LUT-GEMM GEMV (b = 1) over the
OPT-175B fc1 layer (in 12288 -> out 49152, q=3, g=128): x staged into shared
memory, 128 LUTs per slice built, packed planes streamed, scales and offset
applied, cross-slice reduction, fp16 y.  Inputs are
resident in HBM; weights rotate over copies whose total exceeds 3x L2, so
every step streams its weights from HBM (config.l2 says so).

N > 1 (torchrun): strong scaling, tensor parallel (Table 4) --
--tp-mode rows (default): rank r owns fc1 rows [r m/N, (r+1) m/N) and the fp16 rows are
all-gathered; --tp-mode cols: rank r owns fc2 columns [r n/N, (r+1) n/N) and the fp32
partials are all-reduced.  --tp-impl nccl (lutgemm_tp_linear) or p2p (the exchange fused
into the GEMV epilogue over peer memory, lutgemm_p2p_*).  value = whole-layer bytes / step
time (max over ranks); the line adds per-GPU GB/s, the shard GEMV time and the exchange time.

--impl reference times the CPU fp64 oracle (the only reference this paper
has; there is no released code) on rank 0 over a bounded row sample.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LUT-GEMM GEMV us and achieved HBM GB/s (% of B200 peak) at q=3,g=128"
UNIT = "GB/s"


def algorithmic_bytes(m: int, n: int, q: int, g: int, b: int = 1, offset: bool = False, compact: bool = False) -> int:
    """B_alg = m n q/8 (planes) + 2 m (n/g) q (alpha) [+ 2 m (n/g) z] + 2 n b (x) + 2 m b (y);
    the compact uniform format stores one scale s per group instead of q alphas (NEXT-2, has z)."""
    G = n // g
    qa = 1 if compact else q
    return m * n * q // 8 + 2 * m * G * qa + (2 * m * G if (offset or compact) else 0) + 2 * n * b + 2 * m * b


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.005):
        self.samples, self.reasons = [], set()
        self.period = period
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def box_copy_gbs(dev) -> float | None:
    """This box's copy bandwidth, measured as MEASURED_PEAKS.json's hbm_gbs is
    (b.copy_(a) over 1 Gi bf16 elements, read+write bytes, best of 10, CUDA
    events): boxes of the pool differ, so the fraction is also given against it."""
    import torch
    try:
        a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
        b = torch.empty_like(a)
        best = None
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        torch.cuda.empty_cache()
        return 2 * 2 * (1 << 30) / (best * 1e-3) / 1e9
    except Exception:  # noqa: BLE001
        return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_traffic_profile(kernel: str):
    """dram bytes per launch from the committed `ncu --set full` summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def time_oracle(cfg: dict, budget_s: float, min_rows: int = 64, rows_cap: int | None = None):
    """Time the fp64 oracle on a bounded row sample of cfg's layer.
    Returns (GB/s of algorithmic bytes, seconds, rows, threads)."""
    import oracle as O
    from workloads import gen_bcq, gen_x
    m, n, q, g = cfg["m"], cfg["n"], cfg["q"], cfg["g"]
    rows_total = m if rows_cap is None else min(m, rows_cap)
    d = gen_bcq(cfg["seed"], rows_total, n, q, g)
    x = gen_x(cfg["seed"], 1, n)
    t0 = time.perf_counter()
    done = 0
    blk = 1024
    while done < rows_total:
        r = np.arange(done, min(rows_total, done + blk))
        O.bcq_gemv_rows(d["planes"], d["alpha"], None, x, n, g, r)
        done = r[-1] + 1
        if time.perf_counter() - t0 >= budget_s and done >= min_rows:
            break
    dt = time.perf_counter() - t0
    byts = algorithmic_bytes(done, n, q, g)
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # noqa: BLE001
        threads = 1
    return byts / dt / 1e9, dt, int(done), threads


def run_reference(args, cfg) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    from workloads import gen_bcq, gen_x
    m, n, q, g = cfg["m"], cfg["n"], cfg["q"], cfg["g"]
    total_steps = args.steps + args.warmup
    # calibrate rows per step so the whole run ends within ~args.ref_budget seconds
    cal = gen_bcq(cfg["seed"], 256, n, q, g)
    x = gen_x(cfg["seed"], 1, n)
    t0 = time.perf_counter()
    O.bcq_gemv_rows(cal["planes"], cal["alpha"], None, x, n, g, np.arange(256))
    per_row = (time.perf_counter() - t0) / 256
    rows = int(max(4, min(m, args.ref_budget / max(total_steps, 1) / per_row)))
    rows = max(4, rows // 4 * 4)
    d = gen_bcq(cfg["seed"], rows, n, q, g)
    idx = np.arange(rows)
    for _ in range(args.warmup):
        O.bcq_gemv_rows(d["planes"], d["alpha"], None, x, n, g, idx)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.bcq_gemv_rows(d["planes"], d["alpha"], None, x, n, g, idx)
    dt = time.perf_counter() - t0
    byts = algorithmic_bytes(rows, n, q, g)
    value = byts * args.steps / dt / 1e9
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # noqa: BLE001
        threads = 1
    sample = f"fp64 numpy oracle (dequantise then matvec) on the first {rows} of {m} rows of {cfg['name']} per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "m": m, "n": n, "q": q, "g": g, "b": 1, "rows_per_step": rows},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _timed_graph(step, G: int, reps: int, warm: int, stream):
    """Capture G consecutive steps in one CUDA graph; replay `warm` times untimed, then `reps` times
    between CUDA events on `stream`.  Returns (total ms, per-replay ms list)."""
    import torch
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(stream)
    with torch.cuda.graph(graph, stream=cap):
        for i in range(G):
            step(i)
    for _ in range(max(1, warm)):
        graph.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for r in range(reps):
        graph.replay()
        ev[r + 1].record(stream)
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[-1]), [ev[r].elapsed_time(ev[r + 1]) for r in range(reps)], graph


def run_gpu(args, cfg) -> None:
    import torch

    world, rank, local = dist_env()
    if args.same_device:  # validation of the N > 1 path on one GPU: P2P exchange through CUDA IPC, gloo plumbing
        if args.tp_impl != "p2p":
            raise SystemExit("--same-device needs --tp-impl p2p (NCCL refuses two ranks on one GPU)")
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2206_09557_b200 as L
    from workloads import gen_bcq, gen_x

    comm = p2p = None
    cdev = dev  # device of the tensors the process group reduces
    if world > 1:
        import torch.distributed as dist
        if args.same_device:
            dist.init_process_group("gloo")
            cdev = torch.device("cpu")
        else:
            dist.init_process_group("nccl", device_id=dev)
            comm = L.TPComm(rank, world, device=dev)
    mode = args.tp_mode
    m, n, q, g = cfg["m"], cfg["n"], cfg["q"], cfg["g"]
    if mode == "rows":  # m-split: rank r owns rows [r m/N, (r+1) m/N) and sees the full x
        if m % (8 * world):
            raise SystemExit(f"m={m} must split into {world} shards of a multiple of 8 rows")
        ms, ns = m // world, n
    else:  # n-split: rank r owns columns [r n/N, (r+1) n/N) (multiple of g) and x's slice
        if n % (world * g):
            raise SystemExit(f"n={n} must split into {world} shards of whole groups of {g}")
        ms, ns = m, n // world
    d = gen_bcq(cfg["seed"] + 1000 * rank, ms, ns, q, g)  # this rank's shard (seeded per rank)
    x_full = gen_x(cfg["seed"], 1, n)
    x_host = x_full if mode == "rows" else x_full[:, rank * ns:(rank + 1) * ns]
    planes = torch.from_numpy(d["planes"].view(np.int32)).to(dev)
    alpha = torch.from_numpy(d["alpha"]).to(dev)
    B = algorithmic_bytes(m, n, q, g)            # the whole layer (all ranks)
    Bs = algorithmic_bytes(ms, ns, q, g)         # this rank's shard
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    ncopies = max(2, math.ceil(3 * l2 / Bs))
    ws_list = [L.lutgemm_pack_bcq(planes, alpha, None, ns, g) for _ in range(ncopies)]
    del planes, alpha
    x = torch.from_numpy(np.ascontiguousarray(x_host[0])).to(dev)
    y = torch.empty(m, dtype=torch.float16, device=dev)        # full (replicated) output
    y_local = torch.empty(ms, dtype=torch.float16, device=dev)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(ms, ns, 1), dev)
    stream = torch.cuda.current_stream()
    tp_mode = L.TP_ROWS_ALLGATHER if mode == "rows" else L.TP_COLS_ALLREDUCE
    if world > 1:
        tws = L.make_workspace(comm.workspace_bytes(tp_mode, ms, ns, 1), dev) if comm is not None else None
        if args.tp_impl == "p2p":
            p2p = L.P2PGroup(rank, world, rows_out=m if mode == "rows" else 0, cols_m=m if mode == "cols" else 0)

    def step(i):
        w = ws_list[i % ncopies]
        if world == 1:
            L.lutgemm_gemv(w, x, y, ws)
        elif p2p is not None:  # exchange fused into the GEMV epilogue over peer memory (NEXT-1)
            (p2p.gemv_allgather if mode == "rows" else p2p.gemv_allreduce)(w, x, ws, y)
        else:  # GEMV + NCCL collective (lutgemm_tp_linear)
            comm.linear(tp_mode, w, x, y, tws)

    def gemv_only(i):  # the shard's product without the exchange
        L.lutgemm_gemv(ws_list[i % ncopies], x, y_local, ws)

    def barrier():
        if world > 1 and comm is not None:
            comm.wait(stream)  # polls NCCL for asynchronous errors instead of blocking blindly
            torch.distributed.barrier(device_ids=[local])
        elif world > 1:
            torch.cuda.synchronize()
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=cdev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return t.tolist()

    for i in range(max(args.warmup, 3)):
        step(i)
    barrier()
    # the timed region replays a CUDA graph of G consecutive steps (rotating weight copies); PDL
    # edges let each GEMV's weight streaming start under the previous one's tail, as in a
    # decoder's chain of linears
    G = max(ncopies, min(args.steps, 50) // ncopies * ncopies)
    reps = max(1, math.ceil(args.steps / G))
    steps_timed = reps * G
    n0 = L.lutgemm_launch_count()
    sampler = ClockSampler(local, period=float(os.environ.get("LUTGEMM_CLOCK_PERIOD_S", "0.005")))
    barrier()
    with sampler:
        total_ms, per_rep, graph = _timed_graph(step, G, reps, max(1, math.ceil(args.warmup / G)), stream)
    launches_per_step = (L.lutgemm_launch_count() - n0) / G
    del graph
    barrier()
    dist_us = None
    if reps >= 3:
        per = np.array(per_rep) / G * 1e3
        dist_us = {"p10": round(float(np.percentile(per, 10)), 3), "median": round(float(np.median(per)), 3),
                   "p90": round(float(np.percentile(per, 90)), 3), "replays": int(reps), "gemvs_per_replay": int(G)}
    # the shard GEMV alone in the same graph style (TP: exchange cost = step - GEMV)
    gemv_ms = None
    if world > 1:
        barrier()
        gemv_ms, _, gg = _timed_graph(gemv_only, G, reps, 1, stream)
        del gg
    # isolated launches: events around each eager call (no overlap with a neighbour)
    ne = min(args.steps, 200)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ne)]
    barrier()
    for i in range(ne):
        ev[i][0].record(stream)
        step(i)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    iso_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    total_ms, iso_ms, gemv_ms_v = max_over_ranks([total_ms, iso_ms, gemv_ms if gemv_ms is not None else 0.0])
    ms_per_step = total_ms / steps_timed
    value = B / (ms_per_step * 1e-3) / 1e9  # whole-layer bytes over the step time (max over ranks)

    # correctness guard on the timed configuration: sampled rows vs the oracle (every rank's shard)
    parity = None
    if not args.no_check:
        import oracle as O
        step(0)
        torch.cuda.synchronize()
        got_all = y.float().cpu().numpy().astype(np.float64)
        rows_local = np.linspace(0, ms - 1, 64).astype(int)
        if mode == "rows":
            ref = O.bcq_gemv_rows(d["planes"], d["alpha"], None, x_host, ns, g, rows_local)[0]
            got = got_all[rank * ms + rows_local]
            err2, ref2 = float(np.sum((got - ref) ** 2)), float(np.sum(ref ** 2))
        else:  # y = sum over ranks of each shard's partial: sum the fp64 oracle partials across ranks
            part = O.bcq_gemv_rows(d["planes"], d["alpha"], None, x_host, ns, g, rows_local)[0]
            if world > 1:
                t = torch.tensor(part, dtype=torch.float64, device=cdev)
                torch.distributed.all_reduce(t)
                part = t.cpu().numpy()
            got = got_all[rows_local]
            err2, ref2 = float(np.sum((got - part) ** 2)), float(np.sum(part ** 2))
        if world > 1:
            t = torch.tensor([err2, ref2], dtype=torch.float64, device=cdev)
            torch.distributed.all_reduce(t)
            err2, ref2 = float(t[0]), float(t[1])
        parity = math.sqrt(err2 / ref2)

    # e2e through the public API: pinned host x -> device -> product (+ exchange) -> pinned host y
    e2e = None
    xh = torch.from_numpy(np.ascontiguousarray(x_host)).pin_memory()
    yh = torch.empty((1, m), dtype=torch.float16).pin_memory()
    ke = max(10, min(args.steps, 2000))
    if world == 1:
        hws = L.make_workspace(L.lutgemm_host_workspace_bytes(m, n, 1), dev)
        e2e_step = lambda i: L.lutgemm_gemm_host(ws_list[i % ncopies], xh, yh, hws)  # noqa: E731
        api = "lutgemm_gemm_host (C ABI, pinned host buffers, stream-synchronous)"
    else:
        def e2e_step(i):
            x.copy_(xh[0], non_blocking=True)
            step(i)
            yh[0].copy_(y, non_blocking=True)
            stream.synchronize()
        api = (f"H2D x -> {'P2PGroup' if p2p is not None else 'TPComm.linear'} -> D2H y, pinned buffers, "
               "stream-synchronous, every rank")
    for i in range(3):
        e2e_step(i)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(ke):
        e2e_step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    (e_ms,) = max_over_ranks([e0.elapsed_time(e1) / ke])
    e2e = {"value": round(B / (e_ms * 1e-3) / 1e9, 2), "unit": UNIT, "h2d_bytes_per_step": 2 * ns,
           "d2h_bytes_per_step": 2 * m, "us_per_step": round(e_ms * 1e3, 3), "steps": ke, "api": api}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gbs, secs, rows, threads = time_oracle(cfg, budget_s=args.cpu_budget)
        cpu = {"value": round(gbs, 5), "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"fp64 numpy oracle on the first {rows} of {m} rows of {cfg['name']} ({secs:.1f} s)",
               "cpu_model": cpu_model()}

    box = box_copy_gbs(dev) if rank == 0 else None
    if rank == 0:
        peaks = measured_peaks()
        per_gpu = Bs / (ms_per_step * 1e-3) / 1e9  # this rank's shard bytes over the step time
        layer = ("fc1 (OPT-175B FFN-1: in 12288 -> out 49152)" if cfg["name"] == "fc1" else
                 "fc2 (OPT-175B FFN-2: in 49152 -> out 12288)" if cfg["name"] == "fc2" else cfg["name"])
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": steps_timed,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 6), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded uniform random bit-planes, alpha ~ 0.87*2^-i*U(.75,1.25)/sqrt(n), x ~ N(0,1) fp16)",
            "config": {"workload": layer, "m": m, "n": n, "q": q, "g": g, "b": 1,
                       "parallelism": (f"tp{world} {mode} split + {'all-gather' if mode == 'rows' else 'all-reduce'} "
                                       f"({args.tp_impl})" if world > 1 else "single GPU"),
                       "shard": [ms, ns],
                       **({"same_device": "validation run: all ranks on cuda:0 (not a scaling number)"}
                          if args.same_device else {}),
                       "l2": f"{ncopies} rotating weight copies per rank = {ncopies * Bs / 1e6:.0f} MB > 3x L2 "
                             f"({l2 / 1e6:.0f} MB)",
                       "bytes_alg_per_gemv": B},
            "us_per_gemv": round(ms_per_step * 1e3, 3),
            "us_per_gemv_dist": dist_us,
            "pct_of_peak_hbm": round(100 * per_gpu / peaks["hbm_gbs"], 2),
            "roofline": {"bound": "hbm", "achieved": round(per_gpu, 2), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(per_gpu / peaks["hbm_gbs"], 4), "traffic": load_traffic_profile("lut_gemv_kernel"),
                         "kernel": "lut_gemv_kernel (cross-slice reduction fused; one launch per GEMV)",
                         "kernel_us": round(ms_per_step * 1e3, 3),
                         "isolated_us_per_gemv": round(iso_ms * 1e3, 3),
                         "frac_isolated": round(Bs / (iso_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
                         "timing": "CUDA graph of consecutive steps, events around the replays (chain); "
                                   "isolated = events around each eager launch",
                         "peak_source": peaks["source"], "frac_of_nominal_8TBs": round(per_gpu / 8000.0, 4),
                         "box_copy_gbs": None if box is None else round(box, 1),
                         "frac_of_box_copy": None if box is None else round(per_gpu / box, 4)},
            "clocks": sampler.summary(),
            "e2e": e2e,
            "gpu_launches": int(round(launches_per_step * steps_timed)),
            "gpu_launches_per_step": launches_per_step,
            "cpu_baseline": cpu,
            "parity_rel_l2_sampled": parity,
        }
        if world > 1:
            line["tp"] = {"per_gpu_gbs": round(per_gpu, 2), "shard_gemv_us": round(gemv_ms_v / steps_timed * 1e3, 3),
                          "exchange_us": round((total_ms - gemv_ms_v) / steps_timed * 1e3, 3),
                          "impl": args.tp_impl}
        print(json.dumps(line), flush=True)
    if world > 1:
        if p2p is not None:
            p2p.close()
        if comm is not None:
            comm.close()
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="lutgemm", choices=["lutgemm", "reference"])
    ap.add_argument("--config", default=None, help="workload (default fc1; fc2 for --tp-mode cols)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=120.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--tp-mode", default="rows", choices=["rows", "cols"],
                    help="N > 1: rows = m-split + all-gather (fc1); cols = n-split + all-reduce (default config fc2)")
    ap.add_argument("--tp-impl", default="nccl", choices=["nccl", "p2p"],
                    help="N > 1: GEMV + NCCL collective, or the exchange fused into the GEMV epilogue over peer "
                         "memory (NEXT-1; validated with processes sharing one GPU, not yet on NVLink)")
    ap.add_argument("--same-device", action="store_true",
                    help="validation only: every rank on cuda:0, gloo process group, --tp-impl p2p (CUDA IPC)")
    args = ap.parse_args()
    from workloads import CONFIGS
    if args.config is None:
        args.config = "fc2" if args.tp_mode == "cols" else "fc1"
    cfg = dict(CONFIGS[args.config], name=args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
