"""Config 5 in miniature: a 2-layer OPT-175B linear stack (the 4 real layer
shapes) captured in one CUDA graph; layers 0 and 1 checked on sampled rows
against the fp64 oracle (tools/stack.py --check)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_layer_stack_parity_and_timing():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stack.py"), "--layers", "2", "--tokens", "3",
                          "--check"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["finite"]
    assert len(d["parity_rel_l2_sampled"]) == 8
    assert max(d["parity_rel_l2_sampled"].values()) <= 2e-3
    assert d["ms_per_token"] > 0


def _stack_json(out):
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def test_two_layer_stack_p2p_world1():
    """The stack with the fused column-split exchange (NEXT-1) in its CUDA graph at world 1."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stack.py"), "--layers", "2", "--tokens", "3",
                          "--check", "--tp-impl", "p2p"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _stack_json(out)
    assert d["finite"] and d["tp_impl"] == "p2p"
    assert len(d["parity_rel_l2_sampled"]) == 12  # 8 shard checks + 4 TP-output checks (out, fc2 x 2 layers)
    assert max(d["parity_rel_l2_sampled"].values()) <= 2e-3


@pytest.mark.parametrize("nproc", [2, 4])
def test_two_layer_stack_p2p_multi_process_same_gpu(nproc):
    """TP stack (QKV / fc1 by rows, out / fc2 by columns with the fused exchange) with nproc processes
    sharing the GPU through CUDA IPC, one CUDA graph per rank; layers 0 and 1 oracle-checked."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29610 + nproc), os.path.join(ROOT, "tools", "stack.py"),
           "--layers", "2", "--tokens", "3", "--check", "--tp-impl", "p2p", "--same-device"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, (out.stdout + out.stderr)[-3000:]
    d = _stack_json(out)
    assert d["finite"] and d["tp"] == nproc
    assert len(d["parity_rel_l2_sampled"]) == 12
    assert max(d["parity_rel_l2_sampled"].values()) <= 2e-3


@pytest.mark.parametrize("nproc", [1, 2])
def test_two_layer_stack_allgather_scheme(nproc):
    """The contrast variant of SURVEY 8(e): every linear split by rows, y all-gathered through the fused
    exchange (4 per layer); every linear's gathered output checked at this rank's rows against the oracle."""
    script = [os.path.join(ROOT, "tools", "stack.py"), "--layers", "2", "--tokens", "3", "--check", "--tp-impl", "p2p",
              "--tp-scheme", "allgather"]
    if nproc == 1:
        cmd = [sys.executable] + script
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", str(29620 + nproc)] + script + ["--same-device"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, (out.stdout + out.stderr)[-3000:]
    d = _stack_json(out)
    assert d["finite"] and d["tp"] == nproc and d["tp_scheme"] == "allgather"
    assert len(d["parity_rel_l2_sampled"]) == 16  # 8 shard checks + 8 gathered-output checks
    assert max(d["parity_rel_l2_sampled"].values()) <= 2e-3
    if nproc > 1:
        assert d["allgathers_per_token"] == 8
