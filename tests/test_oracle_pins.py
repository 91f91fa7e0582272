"""Pins for the CPU oracle (``-m "not gpu"``): the oracle is checked against
what the paper and mathematics fix -- printed values (Eq. 1 worked example,
Table 5, Sec. 4.1's "2.6x"), closed forms (App. C, Eq. 2, Eq. 4), special
cases and brute force on tiny inputs -- never against itself.

The independent packer used here is ``np.packbits(..., bitorder="little")``,
which shares nothing with ``oracle.pack_signs`` / ``oracle.unpack_signs``.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def indep_pack(signs):
    """Independent canonical packer: +-1 [q][m][n] -> uint32 [q][m][ceil(n/32)]."""
    signs = np.asarray(signs)
    q, m, n = signs.shape
    nw = (n + 31) // 32
    bits = np.zeros((q, m, nw * 32), dtype=np.uint8)
    bits[:, :, :n] = (signs == 1)
    by = np.packbits(bits, axis=-1, bitorder="little")
    return by.view("<u4").reshape(q, m, nw)


# ---------------------------------------------------------------------------
# Eq. 1 worked example
# ---------------------------------------------------------------------------

def test_eq1_worked_example_product(golden_dir):
    ex = _load(golden_dir, "eq1_worked_example.json")
    B = np.array(ex["B"])[None]                     # q = 1
    x = np.array(ex["x"], dtype=np.float64)
    m, n = B.shape[1:]
    planes = indep_pack(B)
    alpha = np.ones((m, 1, 1))
    y = O.bcq_gemv(planes, alpha, None, x, n=n, g=n)[0]
    assert y.tolist() == ex["y"]
    y3 = O.lut_gemv(planes, alpha, None, x, n=n, g=n, mu=ex["mu"])[0]
    assert y3.tolist() == ex["y"]
    # mu = 8 with n padded to 8 columns (x7 = x8 = 0, bits 0): same y (R13)
    B8 = np.concatenate([B, -np.ones((1, m, 2), dtype=int)], axis=-1)
    x8 = np.concatenate([x, [0.0, 0.0]])
    y8 = O.lut_gemv(indep_pack(B8), alpha, None, x8, n=8, g=8, mu=8)[0]
    assert y8.tolist() == ex["y"]


def test_eq1_keys_and_repetition(golden_dir):
    ex = _load(golden_dir, "eq1_worked_example.json")
    B = np.array(ex["B"])[None]
    keys = O.lut_keys(indep_pack(B), n=B.shape[2], mu=ex["mu"])[0]   # [m][t]
    assert keys.T.tolist() == ex["keys_lsb_first"]
    for claim in ex["repeat_claims"]:
        assert int((keys[:, claim["chunk"]] == claim["key"]).sum()) == claim["count"]
    # and the repeated partial sum is what the LUT returns for that key
    T = O.build_luts(np.array(ex["x"], float), mu=3)
    assert T[0][3] == 1 + 2 - 3          # (x1 + x2 - x3)
    assert T[1][4] == -4 - 5 + 6         # (-x4 - x5 + x6)


# ---------------------------------------------------------------------------
# Packing (canonical layout)
# ---------------------------------------------------------------------------

def test_pack_examples(golden_dir):
    ex = _load(golden_dir, "spec_examples.json")["pack"]
    w = O.pack_signs(np.array(ex[0]["row"])[None, None])
    assert int(w[0, 0, 0]) == ex[0]["word"]
    w = O.pack_signs(np.ones((1, 1, ex[1]["row_all_plus_n"]), dtype=int))
    assert int(w[0, 0, 0]) == ex[1]["word"]


@pytest.mark.parametrize("n", [1, 7, 8, 31, 32, 33, 100])
def test_pack_matches_independent_packer_and_round_trips(n):
    rng = np.random.default_rng(n)
    s = rng.choice([-1, 1], size=(3, 5, n))
    p = O.pack_signs(s)
    assert np.array_equal(p, indep_pack(s))
    assert np.array_equal(O.unpack_signs(p, n), s)


def test_exhaustive_round_trip_n8():
    s = np.array(list(itertools.product([-1, 1], repeat=8)))[None]     # 256 rows
    assert np.array_equal(O.unpack_signs(O.pack_signs(s), 8), s)


def test_padding_bits_ignored():
    rng = np.random.default_rng(3)
    s = rng.choice([-1, 1], size=(2, 4, 40))
    p = indep_pack(s)
    p2 = p.copy()
    p2[:, :, -1] |= np.uint32(0xFFFFFF00)            # garbage beyond column 40
    a = rng.random((4, 1, 2))
    x = rng.standard_normal(40)
    assert np.array_equal(O.bcq_gemv(p, a, None, x, 40, 40), O.bcq_gemv(p2, a, None, x, 40, 40))


# ---------------------------------------------------------------------------
# Extended BCQ reconstruction and product (Eq. 3; group-wise P:L296)
# ---------------------------------------------------------------------------

def test_dequantize_examples(golden_dir):
    for ex in _load(golden_dir, "spec_examples.json")["dequantize"]:
        s = np.array(ex["signs"]).reshape(ex["q"], 1, 1)
        w = O.dequantize(indep_pack(s), np.array(ex["alpha"]).reshape(1, 1, -1),
                         np.array([[ex["z"]]]), n=1, g=1)
        assert w[0, 0] == ex["w"]


def test_bias_example(golden_dir):
    ex = _load(golden_dir, "spec_examples.json")["bias"][0]
    n = len(ex["x"])
    planes = indep_pack(np.ones((1, 1, n), dtype=int))
    y = O.bcq_gemv(planes, np.array([[[ex["alpha"]]]]), np.array([[ex["z"]]]),
                   np.array(ex["x"], float), n=n, g=n)
    assert y[0, 0] == ex["y"]


@pytest.mark.parametrize("m,n,q,g,offset", [(5, 40, 2, 8, True), (7, 64, 3, 32, False),
                                            (3, 96, 4, 96, True), (4, 33, 1, 11, True)])
def test_product_against_source_matrices(m, n, q, g, offset):
    """Build W directly from the +-1 source arrays (before packing) and the
    scales; the oracle, fed the independently packed words, must reproduce
    W @ x (catches bit order, plane order, group index, transposes)."""
    rng = np.random.default_rng(m * n + q)
    G = (n + g - 1) // g
    s = rng.choice([-1, 1], size=(q, m, n))
    a = rng.uniform(0.5, 1.5, size=(m, G, q))
    z = rng.standard_normal((m, G)) if offset else None
    X = rng.standard_normal((2, n))
    W = np.zeros((m, n))
    for r in range(m):
        for c in range(n):
            W[r, c] = sum(a[r, c // g, i] * s[i, r, c] for i in range(q)) + (z[r, c // g] if offset else 0.0)
    Y = O.bcq_gemv(indep_pack(s), a, z, X, n=n, g=g)
    np.testing.assert_allclose(Y, X @ W.T, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(O.dequantize(indep_pack(s), a, z, n, g), W, rtol=0, atol=1e-15)


def test_one_hot_probe_decodes_bits():
    """x = e_c with alpha_i = 2^i, z = 0: y_r = sum_i 2^i * b_i[r][c], an odd
    integer that decodes every bit of column c (exact)."""
    rng = np.random.default_rng(11)
    q, m, n = 3, 6, 64
    s = rng.choice([-1, 1], size=(q, m, n))
    a = np.broadcast_to(2.0 ** np.arange(q), (m, 1, q)).copy()
    for c in [0, 5, 31, 32, 63]:
        x = np.zeros(n)
        x[c] = 1.0
        y = O.bcq_gemv(indep_pack(s), a, None, x, n, n)[0]
        expect = sum((2 ** i) * s[i, :, c] for i in range(q))
        assert np.array_equal(y, expect)


def test_linearity_and_scale_equivariance():
    rng = np.random.default_rng(5)
    q, m, n, g = 3, 16, 128, 32
    p = indep_pack(rng.choice([-1, 1], size=(q, m, n)))
    a = rng.random((m, n // g, q))
    z = rng.standard_normal((m, n // g))
    x1, x2 = rng.standard_normal(n), rng.standard_normal(n)
    y = lambda x, aa=a, zz=z: O.bcq_gemv(p, aa, zz, x, n, g)[0]
    np.testing.assert_allclose(y(2.5 * x1 - x2), 2.5 * y(x1) - y(x2), rtol=1e-12, atol=1e-12)
    assert np.array_equal(y(x1, 2 * a, 2 * z), 2 * y(x1))        # power-of-two scaling is exact


# ---------------------------------------------------------------------------
# LUT formulation (App. B)
# ---------------------------------------------------------------------------

def test_build_luts_example(golden_dir):
    ex = _load(golden_dir, "spec_examples.json")["build_luts"][0]
    T = O.build_luts(np.array(ex["x"], float), mu=ex["mu"])
    assert T[0].tolist() == ex["table"]


def test_build_luts_brute_force_and_identities():
    rng = np.random.default_rng(8)
    x = rng.standard_normal(16).astype(np.float16).astype(np.float64)
    T = O.build_luts(x, mu=8)
    assert T.shape == (2, 256)
    for t in range(2):
        for k in range(256):
            bf = 0.0
            for j in range(8):
                bf += (x[8 * t + j] if (k >> j) & 1 else -x[8 * t + j])
            assert T[t, k] == bf                       # fp16 inputs: exact in fp64
        for k in range(256):
            assert T[t, 255 - k] == -T[t, k]           # complement identity
        assert T[t, 255] == x[8 * t:8 * t + 8].sum() and T[t, 0] == -x[8 * t:8 * t + 8].sum()


def test_lut_partials_equal_brute_force_exactly():
    """Every per-(row, group, plane) LUT partial equals the brute-force signed
    sum exactly in fp64 for fp16 activations."""
    rng = np.random.default_rng(21)
    q, m, n, g = 3, 8, 96, 32
    s = rng.choice([-1, 1], size=(q, m, n))
    x = rng.standard_normal(n).astype(np.float16).astype(np.float64)
    a = rng.random((m, n // g, q))
    _, parts = O.lut_gemv(indep_pack(s), a, None, x, n, g, return_partials=True)
    P = parts[0]
    for r in range(m):
        for grp in range(n // g):
            for i in range(q):
                bf = 0.0
                for c in range(grp * g, (grp + 1) * g):
                    bf += s[i, r, c] * x[c]
                assert P[r, grp, i] == bf


@pytest.mark.parametrize("offset", [False, True])
def test_lut_form_matches_definition_on_tiny_config(offset):
    from workloads import gen_bcq, gen_x
    d = gen_bcq(101, 512, 512, 3, 128, offset=offset)
    X = gen_x(101, 3, 512)
    y_def = O.bcq_gemv(d["planes"], d["alpha"], d["offset"], X, 512, 128)
    y_lut = O.lut_gemv(d["planes"], d["alpha"], d["offset"], X, 512, 128)
    np.testing.assert_allclose(y_lut, y_def, rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------------------
# Uniform -> BCQ (App. C)
# ---------------------------------------------------------------------------

def test_uniform_to_bcq_spec_examples(golden_dir):
    for ex in _load(golden_dir, "spec_examples.json")["uniform_to_bcq"]:
        planes, alpha, z = O.uniform_to_bcq(np.array([[ex["code"]]]), np.array([[ex["s"]]]),
                                            np.array([[ex["zhat"]]]), ex["q"])
        assert alpha[0, 0].tolist() == ex["alpha"] and z[0, 0] == ex["z"]
        assert O.dequantize(planes, alpha, z, n=1, g=1)[0, 0] == ex["w"]


@pytest.mark.parametrize("q", [1, 2, 3, 4])
def test_uniform_to_bcq_exact_exhaustive(q):
    """Sum alpha_i b_i + z == s * code + z_hat exactly in fp64, every code,
    2000 random fp16 (s, z_hat) per q (the App. C identity)."""
    rng = np.random.default_rng(100 + q)
    ncode = 2 ** q
    R = 2000
    s = rng.uniform(2.0 ** -13, 4.0, size=(R, 1)).astype(np.float16)
    zh = rng.uniform(-4.0, 4.0, size=(R, 1)).astype(np.float16)
    codes = np.tile(np.arange(ncode), (R, 1))
    planes, alpha, z = O.uniform_to_bcq(codes, s, zh, q)
    w_bcq = O.dequantize(planes, alpha, z, n=ncode, g=ncode)
    w_uni = O.uniform_dequantize(codes, s, zh, g=ncode)
    assert np.array_equal(w_bcq, w_uni)
    # direct closed form of Eq. 6 for a few entries, written with the bits
    for r in range(3):
        for code in range(ncode):
            bh = [(code >> i) & 1 for i in range(q)]
            w6 = float(s[r, 0]) * sum(2 ** i * bh[i] for i in range(q)) + float(zh[r, 0])
            assert w_bcq[r, code] == w6


def test_uniform_path_product():
    from workloads import gen_uniform, gen_x
    d = gen_uniform(404, 64, 256, 4, 128)
    x = gen_x(404, 2, 256)
    planes, alpha, z = O.uniform_to_bcq(d["codes"], d["scale"], d["zero"], 4)
    y_bcq = O.bcq_gemv(planes, alpha, z, x, 256, 128)
    W = O.uniform_dequantize(d["codes"], d["scale"], d["zero"], 128)
    np.testing.assert_allclose(y_bcq, x.astype(np.float64) @ W.T, rtol=1e-13, atol=1e-15)


def test_store_fp16_round_to_nearest_even():
    v = O.store_fp16([1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, 2.0 ** -14 * 1.5])
    assert v.tolist() == [1.0, 1 + 2.0 ** -9, 2.0 ** -14 * 1.5]


# ---------------------------------------------------------------------------
# Closed forms: Eq. 2 op counts, Eq. 4 footprint, Table 5 sizes
# ---------------------------------------------------------------------------

def test_eq2_counts(golden_dir):
    for c in _load(golden_dir, "eq2_counts.json")["cases"]:
        oc = O.op_counts(c["m"], c["n"], c["q"], c["mu"])
        for k in ("c_build", "c_read", "dense_macs"):
            if k in c:
                assert oc[k] == c[k]
        if "paper_reduction_printed" in c:
            red = oc["dense_macs"] / oc["c_read"]
            assert red == c["mu"] / c["q"]                          # q/mu saving, Eq. 2
            assert int(red * 10) / 10 == c["paper_reduction_printed"]


def test_eq4_closed_form():
    for (m, n, q, g) in [(12288, 12288, 3, 128), (49152, 12288, 2, 32), (64, 256, 4, 64)]:
        S = O.memory_footprint_bits(m, n, q, g)["S"]
        assert S * g == m * n * q * (g + 16)                        # m n q (1 + 16/g)


def test_table5_sizes(golden_dir):
    t5 = _load(golden_dir, "table5_opt175b.json")
    L, lin = t5["layers"], t5["linears"]
    dense_bits = L * sum(16 * m * n for m, n in lin)
    for row in t5["rows"]:
        if row["q"] == 16:
            bits = dense_bits
        else:
            bits = L * sum(O.memory_footprint_bits(m, n, row["q"], n if row["g"] == "rowwise" else row["g"],
                                                   scales_per_group=1)["S"] for m, n in lin)
        assert round(bits / 8 / 1e9, 1) == row["size_gb"]
        assert round(dense_bits / bits, 2) == row["ratio"]
