"""GPU parity of the LUT-GEMM path against the fp64 CPU oracle, through the
C ABI (ctypes binding).  Exact probes decode keys / bit order / groups /
offset bit-exactly; metamorphic checks are bitwise; products are checked at
the north_star tolerances (rel-L2 <= 2e-3, max elementwise rel <= 1e-2)."""
import numpy as np
import pytest
import torch

import oracle as O
from tests._helpers import assert_parity, oracle_rows_parallel, parity, stratified_rows
from workloads import CONFIGS, gen_bcq, gen_uniform, gen_x

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def pack(d):
    import paper_2206_09557_b200 as L
    return L.lutgemm_pack_bcq(dev(d["planes"].view(np.int32)), dev(d["alpha"]),
                              None if d["offset"] is None else dev(d["offset"]), d["n"], d["g"])


def run(w, X, f32=False):
    import paper_2206_09557_b200 as L
    Xd = dev(np.atleast_2d(X))
    if Xd.shape[0] == 1 and not f32:
        y = L.lutgemm_gemv(w, Xd[0])[None]
    else:
        y = L.lutgemm_gemm_batched(w, Xd, f32=f32)
    torch.cuda.synchronize()
    return y.float().cpu().numpy().astype(np.float64)


# ---------------------------------------------------------------------------
# exact probes (keys, bit order, plane order, groups, offset)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("q", [1, 3, 4, 8])
def test_one_hot_probe_decodes_every_bit(q):
    """x = e_c, alpha_i = 2^i, z = 0  ->  y_r = sum_i 2^i b_i[r][c] exactly."""
    m, n, g = 64, 2048 + 64, 32
    d = gen_bcq(900 + q, m, n, q, g)
    d["alpha"] = np.broadcast_to((2.0 ** np.arange(q)).astype(np.float16), (m, n // g, q)).copy()
    w = pack(d)
    signs = O.unpack_signs(d["planes"], n).astype(np.int64)
    cols = [0, 1, 7, 8, 31, 32, 255, 256, 1023, 1024, 1031, 2047, 2048, n - 1]
    X = np.zeros((len(cols), n), dtype=np.float16)
    for k, c in enumerate(cols):
        X[k, c] = 1.0
    for b0 in range(0, len(cols), 8):
        Xb = X[b0:b0 + 8]
        Y = run(w, Xb)
        for k in range(Xb.shape[0]):
            c = cols[b0 + k]
            expect = sum((2 ** i) * signs[i, :, c] for i in range(q))
            assert np.array_equal(Y[k], expect.astype(np.float64)), (q, c)
        y1 = run(w, Xb[0])
        assert np.array_equal(y1[0], Y[0])


def test_group_probe():
    """alpha[r][grp][i] = 2^i * (grp+1) for a one-hot x in group grp."""
    m, n, q, g = 32, 1024, 2, 128
    d = gen_bcq(77, m, n, q, g)
    G = n // g
    d["alpha"] = ((2.0 ** np.arange(q))[None, None, :] * (np.arange(G) + 1)[None, :, None]
                  * np.ones((m, 1, 1))).astype(np.float16)
    w = pack(d)
    signs = O.unpack_signs(d["planes"], n).astype(np.int64)
    for c in [5, 130, 300, 777, 1000]:
        x = np.zeros(n, dtype=np.float16)
        x[c] = 1
        y = run(w, x)[0]
        expect = sum((2 ** i) * (c // g + 1) * signs[i, :, c] for i in range(q))
        assert np.array_equal(y, expect.astype(np.float64))


def test_offset_probe():
    """alpha = 0, z = 1, x = [1, 2, 3, ...] -> y_r = sum over groups of x."""
    m, n, q, g = 16, 256, 3, 64
    d = gen_bcq(5, m, n, q, g, offset=True)
    d["alpha"][:] = 0
    d["offset"][:] = 1
    x = (np.arange(n) % 16 + 1).astype(np.float16)
    y = run(pack(d), x)[0]
    assert np.array_equal(y, np.full(m, float(x.astype(np.float64).sum())))


# ---------------------------------------------------------------------------
# metamorphic and determinism (bitwise; requires the fixed-order reduction)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("b", [1, 4])
def test_metamorphic_and_deterministic(b):
    m, n, q, g = 1000, 3072, 3, 128
    d = gen_bcq(31, m, n, q, g, offset=True)
    X = gen_x(31, b, n)
    w = pack(d)
    y = run(w, X, f32=True)
    assert np.array_equal(run(w, X, f32=True), y)                    # bitwise reproducible
    assert np.array_equal(run(w, (2 * X.astype(np.float32)).astype(np.float16), f32=True), 2 * y)
    d2 = dict(d, alpha=(2 * d["alpha"].astype(np.float32)).astype(np.float16),
              offset=(2 * d["offset"].astype(np.float32)).astype(np.float16))
    assert np.array_equal(run(pack(d2), X, f32=True), 2 * y)


# ---------------------------------------------------------------------------
# parity vs the fp64 oracle
# ---------------------------------------------------------------------------

def test_tiny_config_full_parity():
    c = CONFIGS["tiny"]
    d = gen_bcq(c["seed"], c["m"], c["n"], c["q"], c["g"])
    X = gen_x(c["seed"], 1, c["n"])
    y = run(pack(d), X)
    ref = O.bcq_gemv(d["planes"], d["alpha"], None, X, c["n"], c["g"])
    assert_parity(y, ref, "tiny")
    # the LUT formulation of the oracle agrees too
    assert_parity(y, O.lut_gemv(d["planes"], d["alpha"], None, X, c["n"], c["g"]), "tiny-lut")


@pytest.mark.parametrize("m,n,q,g,off", [(1, 32, 1, 32, False), (5, 1056, 3, 32, True), (999, 4096, 2, 64, False),
                                         (777, 5120, 4, 128, True), (300, 2560, 5, 2560, True),
                                         (64, 8192, 8, 256, False), (2049, 1024, 3, 1024, True)])
def test_gemv_shapes_full_parity(m, n, q, g, off):
    d = gen_bcq(m + n + q, m, n, q, g, offset=off)
    X = gen_x(m + n, 1, n)
    y = run(pack(d), X)
    assert_parity(y, O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g), (m, n, q, g))


@pytest.mark.parametrize("b", [2, 3, 4, 5, 8, 16, 31, 32])
@pytest.mark.parametrize("m,n,q,g,off", [(333, 1536, 3, 128, True), (1030, 4096, 2, 32, False),
                                         (64, 2048, 6, 2048, True), (2500, 5152, 1, 32, True)])
def test_batched_full_parity(b, m, n, q, g, off):
    d = gen_bcq(b * 13 + m, m, n, q, g, offset=off)
    X = gen_x(b + m, b, n)
    w = pack(d)
    ref = O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g)
    assert_parity(run(w, X), ref, ("batched", b, m, n))
    # the fp32-output variant (TP column-split partial) agrees as well
    assert_parity(run(w, X, f32=True), ref, ("batched-f32", b))
    # row beta of a batch equals the single-vector result within rounding
    y1 = run(w, X[b - 1])
    assert parity(y1[0], ref[b - 1])["rel_l2"] <= 2e-3


def _sampled_rows(m, seed, k=192):
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(m, size=min(k, m), replace=False).tolist())
    rows |= {0, 1, 2, 3, 255, 256, m - 4, m - 3, m - 2, m - 1}
    return np.array(sorted(r for r in rows if 0 <= r < m))


@pytest.mark.parametrize("name", ["fc1", "fc2"])
def test_full_size_gemv_all_rows(name):
    """BASELINE config 3 at full size, b = 1, in the launch configuration bench.py times: EVERY
    output row against the fp64 oracle (row blocks evaluated in parallel worker processes)."""
    c = CONFIGS[name]
    d = gen_bcq(c["seed"], c["m"], c["n"], c["q"], c["g"])
    X = gen_x(c["seed"], 1, c["n"])
    y = run(pack(d), X)
    ref = oracle_rows_parallel(d["planes"], d["alpha"], None, X, c["n"], c["g"])
    p = assert_parity(y, ref, name)
    print(f"{name} all {c['m']} rows: {p}")


@pytest.mark.parametrize("b", [2, 4, 8, 16])
@pytest.mark.parametrize("name", ["fc1", "fc2"])
def test_ffn_batched_stratified_rows(name, b):
    """Config 3 batched at full size: 4 rows from every 256-row block (every reducer range and
    row block of the batched kernels) against the fp64 oracle, every batch row."""
    c = CONFIGS[name]
    d = gen_bcq(c["seed"], c["m"], c["n"], c["q"], c["g"])
    X = gen_x(c["seed"] + b, b, c["n"])
    Y = run(pack(d), X)
    rows = stratified_rows(c["m"], per_block=4, seed=b)
    ref = oracle_rows_parallel(d["planes"], d["alpha"], None, X, c["n"], c["g"], rows, block=128)
    for beta in range(b):
        assert_parity(Y[beta, rows], ref[beta], (name, b, beta))
    assert_parity(Y[:, rows].ravel(), ref.ravel(), (name, b))


@pytest.mark.parametrize("name", ["attn"])
def test_full_size_gemv_sampled_rows(name):
    """BASELINE full sizes, in the launch configuration bench.py times."""
    c = CONFIGS[name]
    d = gen_bcq(c["seed"], c["m"], c["n"], c["q"], c["g"])
    X = gen_x(c["seed"], 1, c["n"])
    y = run(pack(d), X)[0]
    rows = _sampled_rows(c["m"], c["seed"])
    ref = O.bcq_gemv_rows(d["planes"], d["alpha"], None, X, c["n"], c["g"], rows)[0]
    assert_parity(y[rows], ref, name)
    assert np.all(np.isfinite(y))


@pytest.mark.parametrize("q", [1, 2, 3, 4])
@pytest.mark.parametrize("g", [32, 64, 128, 12288])
def test_attention_qg_grid_sampled(q, g):
    """Config 2: 12288 x 12288, q in {1..4} x g in {32, 64, 128, n}."""
    m = n = 12288
    d = gen_bcq(2000 + 10 * q + g, m, n, q, g)
    X = gen_x(2000 + q, 1, n)
    y = run(pack(d), X)[0]
    rows = _sampled_rows(m, q * g, k=64)
    assert_parity(y[rows], O.bcq_gemv_rows(d["planes"], d["alpha"], None, X, n, g, rows)[0], (q, g))


@pytest.mark.parametrize("compact", [False, True])
@pytest.mark.parametrize("name", ["llama_sq", "llama_up", "llama_down"])
def test_llama_uniform_sampled(name, compact):
    """Config 4: uniform 4-bit codes converted to BCQ with offset (App. C);
    compact: one stored s per group, alpha_i = 2^(i-1) s derived in-kernel."""
    import paper_2206_09557_b200 as L
    c = CONFIGS[name]
    u = gen_uniform(c["seed"], c["m"], c["n"], c["q"], c["g"])
    X = gen_x(c["seed"], 1, c["n"])
    w = L.lutgemm_pack_uniform(dev(u["codes"]), dev(u["scale"]), dev(u["zero"]), c["q"], c["g"], compact=compact)
    y = run(w, X)[0]
    rows = _sampled_rows(c["m"], c["seed"], k=128)
    planes, alpha, z = O.uniform_to_bcq(u["codes"][rows], u["scale"][rows], u["zero"][rows], c["q"])
    ref = O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(z), X, c["n"], c["g"])[0]
    assert_parity(y[rows], ref, name)
    # against the uniform matrix itself: this adds the fp16 storage error of z
    # (R17) to the kernel error, so only the aggregate rel-L2 bar applies here
    W = O.uniform_dequantize(u["codes"][rows], u["scale"][rows], u["zero"][rows], c["g"])
    assert parity(y[rows], (X.astype(np.float64) @ W.T)[0])["rel_l2"] <= 2e-3


def test_fc1_batched_32_sampled():
    c = CONFIGS["fc1"]
    d = gen_bcq(c["seed"], c["m"], c["n"], c["q"], c["g"])
    X = gen_x(c["seed"], 32, c["n"])
    Y = run(pack(d), X)
    rows = stratified_rows(c["m"], per_block=1, seed=7)
    ref = oracle_rows_parallel(d["planes"], d["alpha"], None, X, c["n"], c["g"], rows, block=64)
    assert_parity(Y[:, rows], ref, "fc1-b32")


# ---------------------------------------------------------------------------
# the end-to-end host-buffer entry point and error paths
# ---------------------------------------------------------------------------

def test_host_entry_point_matches_device_path():
    import paper_2206_09557_b200 as L
    m, n, q, g = 4096, 4096, 3, 128
    d = gen_bcq(3, m, n, q, g)
    w = pack(d)
    for b in (1, 2, 4, 8):
        X = gen_x(3, b, n)
        Xh = torch.from_numpy(X).pin_memory()
        # pinned Y: the epilogue writes it over the host link; pageable Y: staged and copied back
        for Yh in (torch.empty((b, m), dtype=torch.float16).pin_memory(), torch.empty((b, m), dtype=torch.float16)):
            ws = L.make_workspace(L.lutgemm_host_workspace_bytes(m, n, b), "cuda")
            L.lutgemm_gemm_host(w, Xh, Yh, ws)
            assert np.array_equal(Yh.float().numpy(), run(w, X).astype(np.float32)), (b, Yh.is_pinned())


def test_error_paths_on_device():
    import paper_2206_09557_b200 as L
    d = gen_bcq(1, 64, 256, 3, 128)
    w = pack(d)
    x = torch.zeros(256 + 8, dtype=torch.float16, device="cuda")
    with pytest.raises(L.LutgemmError) as ei:
        L.lutgemm_gemv(w, x[1:257])
    assert ei.value.status == 2
    ws = torch.zeros(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(L.LutgemmError) as ei:
        L.lutgemm_gemv(w, x[:256], ws=ws)
    assert ei.value.status == 3


@pytest.mark.parametrize("b", [1, 2, 4, 7, 32])
@pytest.mark.parametrize("m,n,q,g", [(333, 1536, 3, 128), (1030, 5152, 4, 32), (64, 2048, 2, 2048), (40, 1024, 6, 64)])
def test_uniform_compact_full_parity(b, m, n, q, g):
    """Compact uniform format vs the fp64 oracle of the App. C
    conversion with the fp16-stored z (R17), GEMV and batched; and against the
    expanded (q alphas) packing of the same source within rounding."""
    import paper_2206_09557_b200 as L
    u = gen_uniform(m + n + q + b, m, n, q, g)
    X = gen_x(m + b, b, n)
    src = (dev(u["codes"]), dev(u["scale"]), dev(u["zero"]))
    wc = L.lutgemm_pack_uniform(*src, q, g, compact=True)
    we = L.lutgemm_pack_uniform(*src, q, g)
    planes, alpha, z = O.uniform_to_bcq(u["codes"], u["scale"], u["zero"], q)
    ref = O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(z), X, n, g)
    yc = run(wc, X)
    assert_parity(yc, ref, ("compact", b, m, n, q, g))
    assert parity(yc.ravel(), run(we, X).ravel())["rel_l2"] <= 1e-3
    # bitwise reproducible and exact under x -> 2x
    yf = run(wc, X, f32=True)
    assert np.array_equal(run(wc, X, f32=True), yf)
    assert np.array_equal(run(wc, (2 * X.astype(np.float32)).astype(np.float16), f32=True), 2 * yf)


@pytest.mark.parametrize("reducers", ["1", "64"])
@pytest.mark.parametrize("m,n,q,g,off", [(6000, 4096, 3, 128, False), (2049, 12288, 4, 64, True)])
def test_gemv_reduction_modes(monkeypatch, reducers, m, n, q, g, off):
    """The fused cross-slice reduction with one reducer per row group and with
    every CTA of the group reducing agrees with the oracle, and the two agree bit
    for bit (same fixed slice order, R11) -- whatever the arrival order."""
    d = gen_bcq(m + q, m, n, q, g, offset=off)
    X = gen_x(n, 1, n)
    w = pack(d)
    monkeypatch.setenv("LUTGEMM_GEMV_REDUCERS", reducers)
    y = run(w, X, f32=True)
    for _ in range(3):
        assert np.array_equal(run(w, X, f32=True), y)
    monkeypatch.setenv("LUTGEMM_GEMV_REDUCERS", "64" if reducers == "1" else "1")
    assert np.array_equal(run(w, X, f32=True), y)
    monkeypatch.delenv("LUTGEMM_GEMV_REDUCERS")
    assert_parity(y, O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g), (m, n, q, g, reducers))


@pytest.mark.parametrize("m,n,q,g,off", [(8192, 22016, 4, 128, True), (1500, 15360, 3, 128, False),
                                         (999, 19456, 2, 64, False)])
def test_fused_and_split_paths_agree(monkeypatch, m, n, q, g, off):
    """Slice counts whose fused grid idles 8-20 % of the SMs (S = 22, 15, 19): the fused mode and the
    split-into-148 path with its separate reduction kernel give the same fp32 result bit for bit
    (both sum the slices in order, R11) and match the oracle."""
    d = gen_bcq(m + n + q, m, n, q, g, offset=off)
    X = gen_x(q + n, 1, n)
    w = pack(d)
    y = run(w, X, f32=True)
    monkeypatch.setenv("LUTGEMM_FUSE_MIN_PCT", "101")
    assert np.array_equal(run(w, X, f32=True), y)
    monkeypatch.delenv("LUTGEMM_FUSE_MIN_PCT")
    assert_parity(run(w, X), O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g), (m, n, q, g))


def _random_configs(k=24, seed=2206):
    """Seeded random shapes over the whole supported space: m and n tails, q 1..8, every g kind
    (32..1024 powers of two, multiples of 1024, row-wise), b 1..32, offset / compact uniform."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < k:
        q = int(rng.integers(1, 9))
        n = 32 * int(rng.integers(1, 200))
        kind = rng.integers(0, 3)
        if kind == 0:
            g = int(2 ** rng.integers(5, 11))
        elif kind == 1:
            g = 1024 * int(rng.integers(1, 4))
        else:
            g = n
        if n % g:
            continue
        m = int(rng.integers(1, 3000))
        b = int(rng.choice([1, 1, 2, 3, 4, 8, 13, 32]))
        fmt = int(rng.integers(0, 3))  # 0 BCQ, 1 BCQ + offset, 2 uniform compact
        out.append((m, n, q, g, b, fmt))
    return out


@pytest.mark.parametrize("m,n,q,g,b,fmt", _random_configs())
def test_random_shapes_full_parity(m, n, q, g, b, fmt):
    import paper_2206_09557_b200 as L
    X = gen_x(m + b, b, n)
    if fmt == 2:
        u = gen_uniform(m + n + q, m, n, q, g)
        w = L.lutgemm_pack_uniform(dev(u["codes"]), dev(u["scale"]), dev(u["zero"]), q, g, compact=True)
        planes, alpha, z = O.uniform_to_bcq(u["codes"], u["scale"], u["zero"], q)
        ref = O.bcq_gemv(planes, O.store_fp16(alpha), O.store_fp16(z), X, n, g)
    else:
        d = gen_bcq(m + n + q, m, n, q, g, offset=fmt == 1)
        w = pack(d)
        ref = O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, n, g)
    assert_parity(run(w, X), ref, (m, n, q, g, b, fmt))
