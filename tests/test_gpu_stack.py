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
