"""Fused GEMV + rows all-gather / column all-reduce over peer memory (SURVEY NEXT-1,
lutgemm_p2p_*): world 1 in-process, and 2 / 4 processes sharing the one GPU through
CUDA IPC (the handles travel over gloo).  Every result is checked against the fp64
oracle at the north_star tolerances; in addition the gathered rows must equal the
1-GPU rows bit for bit, over several rounds (both halves of the double buffer)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle as O
from tests._helpers import assert_parity
from workloads import gen_bcq, gen_uniform, gen_x

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_p2p_world1_matches_gemv():
    import paper_2206_09557_b200 as L
    m, n, q, g = 6000, 4096, 3, 128
    d = gen_bcq(3, m, n, q, g)
    w = L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(), torch.from_numpy(d["alpha"]).cuda(),
                           None, n, g)
    grp = L.P2PGroup(0, 1, rows_out=m)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
    for r in range(5):
        x = torch.from_numpy(gen_x(r, 1, n)[0]).cuda()
        y = torch.empty(m, dtype=torch.float16, device="cuda")
        grp.gemv_allgather(w, x, ws, y)
        ref = L.lutgemm_gemv(w, x)
        torch.cuda.synchronize()
        assert_parity(y.float().cpu().numpy(), O.bcq_gemv(d["planes"], d["alpha"], None, gen_x(r, 1, n), n, g),
                      ("p2p rows", r))
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16))
    grp.close()


def test_p2p_allreduce_world1_matches_gemv():
    import paper_2206_09557_b200 as L
    m, n, q, g = 6000, 4096, 3, 128
    d = gen_bcq(5, m, n, q, g)
    w = L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(), torch.from_numpy(d["alpha"]).cuda(),
                           None, n, g)
    grp = L.P2PGroup(0, 1, rows_out=m, cols_m=m)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
    for r in range(5):
        x = torch.from_numpy(gen_x(r, 1, n)[0]).cuda()
        y = torch.empty(m, dtype=torch.float16, device="cuda")
        grp.gemv_allreduce(w, x, ws, y)
        ref = L.lutgemm_gemv(w, x)
        torch.cuda.synchronize()
        assert_parity(y.float().cpu().numpy(), O.bcq_gemv(d["planes"], d["alpha"], None, gen_x(r, 1, n), n, g),
                      ("p2p cols", r))
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16))  # one slot: the fp16 of the same fp32 row
    grp.close()


@pytest.mark.parametrize("compact", [False, True])
@pytest.mark.parametrize("mode", ["allgather", "allreduce"])
def test_p2p_world1_uniform_offset_formats(mode, compact):
    """The epilogue stores under the offset (extended BCQ, App. C) and compact uniform weights."""
    import paper_2206_09557_b200 as L
    m, n, q, g = 4096, 8192, 4, 128
    u = gen_uniform(6, m, n, q, g)
    w = L.lutgemm_pack_uniform(torch.from_numpy(u["codes"]).cuda(), torch.from_numpy(u["scale"]).cuda(),
                               torch.from_numpy(u["zero"]).cuda(), q, g, compact=compact)
    grp = L.P2PGroup(0, 1, rows_out=m, cols_m=m)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(m, n, 1), "cuda")
    planes, alpha, z = O.uniform_to_bcq(u["codes"], u["scale"], u["zero"], q)
    for r in range(3):
        x = torch.from_numpy(gen_x(20 + r, 1, n)[0]).cuda()
        y = torch.empty(m, dtype=torch.float16, device="cuda")
        if mode == "allgather":
            grp.gemv_allgather(w, x, ws, y)
        else:
            grp.gemv_allreduce(w, x, ws, y)
        ref = L.lutgemm_gemv(w, x)
        torch.cuda.synchronize()
        assert_parity(y.float().cpu().numpy(),
                      O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(z), gen_x(20 + r, 1, n), n, g),
                      (mode, compact, r))
        assert torch.equal(y.view(torch.int16), ref.view(torch.int16))
    grp.close()


def test_p2p_rejects_unfused_shapes():
    import paper_2206_09557_b200 as L
    d = gen_bcq(4, 8, 1024, 3, 128)  # 2 row quads < J CTAs per slice: not the fused mode
    w = L.lutgemm_pack_bcq(torch.from_numpy(d["planes"].view(np.int32)).cuda(), torch.from_numpy(d["alpha"]).cuda(),
                           None, 1024, 128)
    grp = L.P2PGroup(0, 1, rows_out=8)
    ws = L.make_workspace(L.lutgemm_workspace_bytes(8, 1024, 1), "cuda")
    with pytest.raises(L.LutgemmError) as ei:
        grp.gemv_allgather(w, torch.zeros(1024, dtype=torch.float16, device="cuda"), ws,
                           torch.empty(8, dtype=torch.float16, device="cuda"))
    assert ei.value.status == 6
    grp.close()


def _run_check(nproc, port, *args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "p2p_check.py"), "--same-device", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    return out


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("mode", ["rows", "cols"])
@pytest.mark.parametrize("nproc", [2, 4])
def test_p2p_multi_process_same_gpu(nproc, mode, graph):
    """nproc processes share the GPU through CUDA IPC; 4 rounds issued back to back without a host
    synchronisation (or captured in a CUDA graph and replayed twice); every rank's result of every
    round against the fp64 oracle, plus bitwise checks (rows: == 1-GPU GEMV; cols: equal across ranks)."""
    port = 29540 + nproc + (10 if mode == "cols" else 0) + (20 if graph else 0)
    out = _run_check(nproc, port, "--rounds", "4", "--mode", mode, *(["--graph"] if graph else []))
    assert out.count(": PASS") == 4 * nproc and ": FAIL" not in out, out[-3000:]


@pytest.mark.parametrize("mode,nproc,rows,cols", [("rows", 4, 1184, 4096), ("cols", 4, 1000, 8192),
                                                   ("cols", 2, 1001, 4096)])
def test_p2p_multi_process_uneven_shapes(mode, nproc, rows, cols):
    """Shards whose rows do not fill the 8-row units and owner blocks evenly: rows 1184 / 4 = 296 per
    rank; cols m = 1000 over 4 owners (blocks 256, 256, 256, 232) and an odd m = 1001 over 2 owners
    (the last LL word carries one real row); column shards of 2048 (2 LUT slices: the fused mode needs
    at least one 8-row unit per CTA).  Back-to-back rounds, every rank against the oracle."""
    port = 29570 + nproc + (10 if mode == "cols" else 0) + (rows % 7)
    out = _run_check(nproc, port, "--rounds", "3", "--mode", mode, "--rows", str(rows), "--cols", str(cols))
    assert out.count(": PASS") == 3 * nproc and ": FAIL" not in out, out[-3000:]


def test_p2p_world1_graph_capture():
    """World 1, both modes: a CUDA graph of rounds replays correctly (device-side round counter)."""
    for mode in ("rows", "cols"):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "p2p_check.py"), "--rounds", "5", "--graph",
                            "--mode", mode], capture_output=True, text=True, timeout=600, cwd=ROOT)
        out = r.stdout + r.stderr
        assert r.returncode == 0 and out.count(": PASS") == 5, out[-3000:]


def test_p2p_dead_peer_traps_instead_of_hanging():
    """Failure detection: a peer that never makes its call makes the waiting rank's fused
    exchange trap after LUTGEMM_P2P_TIMEOUT_MS (here 2 s) -- a loud launch failure, not a GPU hang."""
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LUTGEMM_P2P_TIMEOUT_MS="2000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29641", os.path.join(root, "tools", "p2p_timeout.py")]
    t0 = time.time()
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root, env=env)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-3000:]
    assert "p2p timeout: trapped" in text, text[-3000:]
    assert time.time() - t0 < 240
