"""bench.py keeps the driver's contract: one JSON line with the required keys
(reference arm on CPU here; the GPU arm under -m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "cpu_baseline"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run_bench("--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-budget", "2")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["gpu_launches"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "fc1"


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = run_bench("--steps", "100", "--warmup", "3", "--no-cpu")
    assert BASE_KEYS <= set(d)
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True and d["n_gpus"] == 1
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and r["bound"] == "hbm"
    assert 0 < r["frac"] < 1.2 and r["achieved"] == pytest.approx(d["value"], rel=1e-3)
    assert d["gpu_launches"] >= d["steps"] and d["gpu_launches_per_step"] == 1.0
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 12288 and d["e2e"]["d2h_bytes_per_step"] == 2 * 49152
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["parity_rel_l2_sampled"] < 2e-3


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["rows", "cols"])
def test_tp_arm_two_ranks_same_device(mode):
    """The N > 1 (strong-scaling, tensor-parallel) arm of bench.py with 2 ranks, validated on one GPU:
    --same-device runs both ranks on cuda:0 with the fused P2P exchange over CUDA IPC; the line keeps
    the contract and the sampled rows of the gathered / reduced output match the oracle."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(29650 + (mode == "cols")), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "20", "--warmup", "3", "--no-cpu", "--tp-impl", "p2p", "--tp-mode", mode, "--same-device"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["parity_rel_l2_sampled"] <= 2e-3
    assert d["tp"]["impl"] == "p2p" and "exchange_us" in d["tp"]
    assert d["config"]["shard"] == ([24576, 12288] if mode == "rows" else [12288, 24576])
