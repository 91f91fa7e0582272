"""Multi-process (gloo, world size 2, CPU) checks of the tensor-parallel
partition semantics used by lutgemm_tp_linear:

* m-split: each rank's rows, all-gathered, equal the full product;
* n-split: each rank's column shard (whole groups, with its bias share and
  its x slice), all-reduced, equals the full product.

The per-shard product is the fp64 oracle; the exchange is a real
torch.distributed collective between two processes."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    import oracle as O
    from paper_2206_09557_b200.tp import shard_cols, shard_rows
    from workloads import gen_bcq, gen_x

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    m, n, q, g = 64, 512, 3, 64
    d = gen_bcq(17, m, n, q, g, offset=True)
    X = gen_x(17, 2, n)
    full = O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g)

    p, a, z = shard_rows(d["planes"], d["alpha"], d["offset"], rank, world)
    y_loc = torch.from_numpy(O.bcq_gemv(p, a, z, X, n, g))
    parts = [torch.empty_like(y_loc) for _ in range(world)]
    dist.all_gather(parts, y_loc)
    rows_ok = np.allclose(torch.cat(parts, dim=1).numpy(), full, rtol=1e-12, atol=1e-12)

    p, a, z = shard_cols(d["planes"], d["alpha"], d["offset"], n, g, rank, world)
    ns = n // world
    y_part = torch.from_numpy(O.bcq_gemv(p, a, z, X[:, rank * ns:(rank + 1) * ns], ns, g))
    dist.all_reduce(y_part)
    cols_ok = np.allclose(y_part.numpy(), full, rtol=1e-12, atol=1e-12)
    results[rank] = (rows_ok, cols_ok)
    dist.destroy_process_group()


def test_tp_partition_semantics_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    procs = [ctx.Process(target=_worker, args=(r, world, port, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert dict(results) == {0: (True, True), 1: (True, True)}


def test_shard_ranges_reject_bad_splits():
    from paper_2206_09557_b200.tp import col_range, row_range
    assert row_range(49152, 3, 8) == (18432, 24576)
    assert col_range(49152, 128, 7, 8) == (43008, 49152)
    with pytest.raises(ValueError):
        row_range(10, 0, 4)
    with pytest.raises(ValueError):
        col_range(512, 128, 0, 8)
