"""CPU-only checks of the boundary: the C-ABI library loads, exports every
symbol include/lutgemm.h declares, and its host-side logic (sizes, argument
validation) behaves as documented.  No compute call needs a GPU here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lutgemm.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lutgemm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import paper_2206_09557_b200.lutgemm as B
    lib = ctypes.CDLL(B.LIB_PATH)
    names = _declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding wraps exactly the declared set
    assert sorted(n for n, _, _ in B.SIGNATURES) == names


def test_library_is_sm100a_only():
    import subprocess
    import paper_2206_09557_b200.lutgemm as B
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if "ELF" in line)


def test_product_kernels_fit_the_shared_memory_opt_in():
    """The product kernels size their dynamic shared memory for the LUT; a static __shared__ variable
    on top (beyond the 1 KB the system reserves per CTA) once pushed a 227 KB request past the per-CTA
    opt-in maximum and every launch failed with cudaErrorInvalidValue, so none may declare one."""
    import subprocess
    import paper_2206_09557_b200.lutgemm as B
    out = subprocess.run(["cuobjdump", "-res-usage", B.LIB_PATH], capture_output=True, text=True).stdout
    found = 0
    for name, shared in re.findall(r"Function (\S+):\s*\n\s*REG:\d+ STACK:\d+ SHARED:(\d+)", out):
        if re.search(r"lut_gemv_kernel|lut_gemvv_kernel|lut_gemm_batched_kernel", name):
            found += 1
            assert int(shared) <= 1024, (name, shared)
    assert found >= 45


def test_abi_version_and_sizes():
    import paper_2206_09557_b200 as L
    from paper_2206_09557_b200.lutgemm import lib
    assert lib.lutgemm_abi_version() == 1
    # one record stream: m4*q*n/8 key bytes + m4*(n/g)*q*2 alpha (+ m4*(n/g)*2 z) (layout.cuh)
    assert L.lutgemm_packed_bytes(49152, 12288, 3, 128, False) == 226492416 + 28311552
    assert L.lutgemm_packed_bytes(22013, 8192, 4, 128, True) == 22016 * 4 * 1024 + 22016 * 64 * 4 * 2 + 22016 * 64 * 2
    # row-wise g > 1024: the group's scales repeat in each of the S slices; regions 256-B padded
    assert L.lutgemm_packed_bytes(8, 2048, 3, 2048, False) == 2 * (2 * 1536 + 256)
    # workspace: 2 x 256 u32 group counters + S*b*m4 fp32 split-K partials (256-B rounded)
    assert L.lutgemm_workspace_bytes(49152, 12288, 1) == 2304 + 12 * 49152 * 4
    # b <= 4: sub-slice partials of the GEMV-structured kernel, [V S][b_pad][m4] fp32 (V = 4 for b = 3, 4)
    assert L.lutgemm_workspace_bytes(49152, 12288, 4) == 2304 + 4 * 12 * 4 * 49152 * 4
    assert L.lutgemm_workspace_bytes(5, 1056, 3) == 2304 + (4 * 2 * 4 * 8 * 4 + 255) // 256 * 256
    assert L.lutgemm_workspace_bytes(49152, 12288, 2) == 2304 + 2 * 12 * 2 * 49152 * 4
    # b > 4: room for the vector-slot kernel ([S][b_pad][m4]) and for chunks of <= 4 rows (the b = 4 partials)
    assert L.lutgemm_workspace_bytes(49152, 12288, 8) == 2304 + 4 * 12 * 4 * 49152 * 4
    assert L.lutgemm_workspace_bytes(49152, 12288, 32) == 2304 + 12 * 32 * 49152 * 4


@pytest.mark.parametrize("m,n,q,g", [(0, 64, 3, 32), (8, 64, 0, 32), (8, 64, 9, 32), (8, 96, 3, 64),
                                     (8, 64, 3, 96), (8, 44, 3, 44), (8, 96, 3, 12), (8, 64, 3, 0),
                                     (8, 4, 3, 4), (8, 4104, 3, 32)])
def test_invalid_shapes_rejected(m, n, q, g):
    import paper_2206_09557_b200 as L
    with pytest.raises(L.LutgemmError) as ei:
        L.lutgemm_packed_bytes(m, n, q, g, False)
    assert ei.value.status == 1
    assert "must" in str(ei.value)


@pytest.mark.parametrize("m,n,q,g,off", [(5, 48, 3, 48, False), (8, 64, 3, 16, True), (8, 192, 3, 96, False),
                                         (3, 6144, 3, 1536, True), (9, 4800, 3, 96, True), (6, 4608, 2, 384, False),
                                         (7, 4104, 3, 24, True), (10, 1000, 2, 8, False), (3, 4104, 4, 4104, True),
                                         (4, 12288, 3, 128, False), (2, 2040, 5, 40, True)])
def test_general_shapes_accepted_and_sized(m, n, q, g, off):
    """SURVEY 8(b)'s shape contract (n % 8, g % 8, g | n): accepted, and the library's packed size
    equals the independent numpy statement of the layout (tests/_helpers.native_pack_reference)."""
    import numpy as np
    import paper_2206_09557_b200 as L
    from tests._helpers import native_pack_reference
    from workloads import gen_bcq
    d = gen_bcq(1, m, n, q, g, offset=off)
    ref = native_pack_reference(d["planes"], d["alpha"], d["offset"], m, n, q, g)
    assert L.lutgemm_packed_bytes(m, n, q, g, off) == len(ref)


def test_compact_format_needs_whole_lane_groups():
    import paper_2206_09557_b200 as L
    assert L.lutgemm_packed_bytes(8, 4800, 3, 96, True, L.FMT_UNIFORM_COMPACT) > 0
    with pytest.raises(L.LutgemmError) as ei:
        L.lutgemm_packed_bytes(8, 4104, 3, 24, True, L.FMT_UNIFORM_COMPACT)
    assert ei.value.status == 1 and "compact" in str(ei.value)


def test_gemv_argument_validation_without_gpu():
    """Validation happens before any device work: NULL/misaligned/small-ws
    arguments are rejected on a CPU-only host too."""
    from paper_2206_09557_b200.lutgemm import lib, lutgemm_weight
    w = lutgemm_weight(64, 64, 3, 32, 0, 0, 4096)
    st = lib.lutgemm_gemv(ctypes.byref(w), 4096 + 2, 8192, 16384, 1 << 20, None)
    assert st == 2 and b"x must be 16-byte aligned" in lib.lutgemm_last_error()
    st = lib.lutgemm_gemv(ctypes.byref(w), 4096, 8192, 16384, 16, None)
    assert st == 3 and b"workspace" in lib.lutgemm_last_error()
    st = lib.lutgemm_gemm_batched(ctypes.byref(w), 4096, 33, 8192, 16384, 1 << 20, None)
    assert st == 1
    w.has_offset = 2
    st = lib.lutgemm_gemv(ctypes.byref(w), 4096, 8192, 16384, 1 << 20, None)
    assert st == 1 and b"offset" in lib.lutgemm_last_error()
    w.has_offset, w.data = 0, 4100
    st = lib.lutgemm_gemv(ctypes.byref(w), 4096, 8192, 16384, 1 << 20, None)
    assert st == 2 and b"weight data" in lib.lutgemm_last_error()


def test_p2p_argument_validation_without_gpu():
    """lutgemm_p2p_*: bad arguments are rejected before any CUDA call (status 1 = INVALID_ARG)."""
    import paper_2206_09557_b200.lutgemm as B
    lib = B.lib
    rec = (ctypes.c_uint8 * 256)()
    h = ctypes.c_void_p()
    for rank, world in [(0, 0), (0, 9), (2, 2), (-1, 2)]:
        assert lib.lutgemm_p2p_create(rank, world, 1024, ctypes.byref(h), rec) == 1
    assert lib.lutgemm_p2p_create(0, 1, 0, ctypes.byref(h), rec) == 1   # out_bytes 0
    assert lib.lutgemm_p2p_connect(None, rec) == 1
    w = B.lutgemm_weight()
    assert lib.lutgemm_p2p_gemv_allgather(None, ctypes.byref(w), None, None, 0, None, None) == 1
    assert lib.lutgemm_p2p_gemv_allreduce(None, ctypes.byref(w), None, None, 0, None, None) == 1
    assert lib.lutgemm_p2p_destroy(None) == 0
    # the shard is validated like any weight (shape rule, format, alignment) before the group
    for bad, msg in [((64, 1024, 9, 128, 0, 0, 4096), b"q=9"), ((64, 1024, 3, 96, 0, 0, 4096), b"g=96"),
                     ((64, 1024, 3, 128, 0, 7, 4096), b"format"), ((64, 1024, 3, 128, 0, 0, 4100), b"aligned")]:
        w = B.lutgemm_weight(*bad)
        for fn in (lib.lutgemm_p2p_gemv_allgather, lib.lutgemm_p2p_gemv_allreduce):
            st = fn(None, ctypes.byref(w), 4096, 8192, 1 << 20, None, 16384)
            assert st in (1, 2) and msg in lib.lutgemm_last_error(), (bad, lib.lutgemm_last_error())
    # window sizes: rows = 2 m (256-B rounded); cols = P mb fp32 slots + P mb fp16, mb = 8 ceil(ceil(m/P)/8)
    # LL words: 8 bytes per half2 row pair (rows), per fp32 slot row and per half2 row pair (cols)
    assert lib.lutgemm_p2p_window_bytes(8, B.TP_ROWS_ALLGATHER, 49152) == 49152 * 4
    assert lib.lutgemm_p2p_window_bytes(8, B.TP_COLS_ALLREDUCE, 12288) == 8 * 1536 * 8 + 8 * 1536 * 4
    assert lib.lutgemm_p2p_window_bytes(3, B.TP_COLS_ALLREDUCE, 100) == 1024 + 512  # mb = 40: 960 B + 480 B, 256-B rounded
    assert lib.lutgemm_p2p_window_bytes(9, B.TP_COLS_ALLREDUCE, 100) == 0
