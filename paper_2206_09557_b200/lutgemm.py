"""ctypes binding of liblutgemm.so (include/lutgemm.h) -- argument marshalling only.

Every step of the LUT-GEMM path runs in the CUDA library; this module only
turns PyTorch tensors (device memory, streams) into pointers and sizes.  There
is no CPU fallback: importing this module without the built library raises.
Function names mirror the C ABI.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblutgemm.so")

OK = 0
STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "MISALIGNED", 3: "WORKSPACE", 4: "CUDA", 5: "NCCL", 6: "UNSUPPORTED"}
SRC_BCQ, SRC_UNIFORM, SRC_UNIFORM_COMPACT = 0, 1, 2
FMT_BCQ, FMT_UNIFORM_COMPACT = 0, 1
TP_ROWS_LOCAL, TP_ROWS_ALLGATHER, TP_COLS_ALLREDUCE = 0, 1, 2


class LutgemmError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class lutgemm_weight(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("n", ctypes.c_int32), ("q", ctypes.c_int32), ("g", ctypes.c_int32),
                ("has_offset", ctypes.c_int32), ("format", ctypes.c_int32), ("data", ctypes.c_void_p)]


class lutgemm_pack_src(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("m", ctypes.c_int32), ("n", ctypes.c_int32), ("q", ctypes.c_int32),
                ("g", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("planes", ctypes.c_void_p), ("alpha", ctypes.c_void_p), ("offset", ctypes.c_void_p),
                ("codes", ctypes.c_void_p), ("scale", ctypes.c_void_p), ("zero", ctypes.c_void_p)]


# (name, restype, argtypes) of every symbol include/lutgemm.h declares
_P = ctypes.c_void_p
_SZ = ctypes.c_size_t
_I = ctypes.c_int
SIGNATURES = [
    ("lutgemm_abi_version", _I, []),
    ("lutgemm_last_error", ctypes.c_char_p, []),
    ("lutgemm_source_hash", ctypes.c_char_p, []),
    ("lutgemm_packed_bytes", _I, [_I, _I, _I, _I, _I, ctypes.POINTER(_SZ)]),
    ("lutgemm_packed_bytes_fmt", _I, [_I, _I, _I, _I, _I, _I, ctypes.POINTER(_SZ)]),
    ("lutgemm_pack_bcq", _I, [ctypes.POINTER(lutgemm_pack_src), ctypes.POINTER(lutgemm_weight), _P]),
    ("lutgemm_unpack_bcq", _I, [ctypes.POINTER(lutgemm_weight), _P, _P, _P, _P]),
    ("lutgemm_workspace_bytes", _SZ, [_I, _I, _I]),
    ("lutgemm_workspace_init", _I, [_P, _SZ, _P]),
    ("lutgemm_gemv", _I, [ctypes.POINTER(lutgemm_weight), _P, _P, _P, _SZ, _P]),
    ("lutgemm_gemm_batched", _I, [ctypes.POINTER(lutgemm_weight), _P, _I, _P, _P, _SZ, _P]),
    ("lutgemm_gemm_batched_f32", _I, [ctypes.POINTER(lutgemm_weight), _P, _I, _P, _P, _SZ, _P]),
    ("lutgemm_host_workspace_bytes", _SZ, [_I, _I, _I]),
    ("lutgemm_gemm_host", _I, [ctypes.POINTER(lutgemm_weight), _P, _I, _P, _P, _SZ, _P]),
    ("lutgemm_trace_enable", _I, [_I]),
    ("lutgemm_trace_read", _SZ, [ctypes.POINTER(ctypes.c_uint64), _SZ]),
    ("lutgemm_launch_count", ctypes.c_uint64, []),
    ("lutgemm_p2p_window_bytes", _SZ, [_I, _I, _I]),
    ("lutgemm_p2p_create", _I, [_I, _I, _SZ, ctypes.POINTER(_P), _P]),
    ("lutgemm_p2p_connect", _I, [_P, _P]),
    ("lutgemm_p2p_gemv_allgather", _I, [_P, ctypes.POINTER(lutgemm_weight), _P, _P, _SZ, _P, _P]),
    ("lutgemm_p2p_gemv_allreduce", _I, [_P, ctypes.POINTER(lutgemm_weight), _P, _P, _SZ, _P, _P]),
    ("lutgemm_p2p_destroy", _I, [_P]),
    ("lutgemm_quantize_rtn", _I, [_P, _I, _I, _I, _I, _P, _P, _P, _P]),
    ("lutgemm_quantize_bcq", _I, [_P, _I, _I, _I, _I, _I, _P, _P, _P]),
    ("lutgemm_tp_unique_id", _I, [_P]),
    ("lutgemm_tp_init", _I, [_I, _I, _P, ctypes.POINTER(_P)]),
    ("lutgemm_tp_workspace_bytes", _SZ, [_P, _I, _I, _I, _I]),
    ("lutgemm_tp_linear", _I, [_P, _I, ctypes.POINTER(lutgemm_weight), _P, _I, _P, _P, _SZ, _P]),
    ("lutgemm_tp_destroy", _I, [_P]),
    ("lutgemm_tp_async_error", _I, [_P]),
    ("lutgemm_tp_abort", _I, [_P]),
    ("lutgemm_tp_rank", _I, [_P]),
    ("lutgemm_tp_nranks", _I, [_P]),
]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built (run `python -c 'import __graft_entry__ as g; g.build()'`); "
                          "there is no CPU fallback for the LUT-GEMM path")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        try:
            fn = getattr(lib, name)
        except AttributeError as e:
            raise ImportError(f"{LIB_PATH} lacks {name} (stale build): rebuild with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`") from e
        fn.restype = res
        fn.argtypes = args
    # the library must be the build of the sources next to it (no stale binary)
    if os.path.isdir(os.path.join(_HERE, "csrc")):
        from paper_2206_09557_b200._build import source_hash
        have, want = lib.lutgemm_source_hash().decode(), source_hash()
        if have != want:
            raise ImportError(f"{LIB_PATH} was built from sources {have}, the tree has {want}: rebuild with "
                              "`python -c 'import __graft_entry__ as g; g.build()'`")
    return lib


lib = _load()


def _check(fn: str, status: int):
    if status != OK:
        raise LutgemmError(fn, status, lib.lutgemm_last_error().decode(errors="replace"))


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def lutgemm_packed_bytes(m: int, n: int, q: int, g: int, has_offset: bool, fmt: int = FMT_BCQ) -> int:
    a = _SZ()
    _check("lutgemm_packed_bytes_fmt",
           lib.lutgemm_packed_bytes_fmt(m, n, q, g, int(has_offset), int(fmt), ctypes.byref(a)))
    return a.value


@dataclass
class PackedBCQ:
    """A packed weight resident on the device (kernel-native record stream);
    the torch tensor ``data`` owns the memory, ``struct`` is its C view."""
    m: int
    n: int
    q: int
    g: int
    has_offset: bool
    data: torch.Tensor
    struct: lutgemm_weight = field(default=None)
    fmt: int = FMT_BCQ

    @classmethod
    def empty(cls, m, n, q, g, has_offset, device, fmt: int = FMT_BCQ, out: torch.Tensor | None = None) -> "PackedBCQ":
        nb = lutgemm_packed_bytes(m, n, q, g, has_offset, fmt)
        if out is None:
            data = torch.empty(nb, dtype=torch.uint8, device=device)
        else:  # caller-provided storage (e.g. a view into one arena holding many layers)
            if out.dtype != torch.uint8 or not out.is_cuda or not out.is_contiguous() or out.numel() < nb \
                    or out.data_ptr() % 256:
                raise ValueError(f"out must be a contiguous 256-byte aligned CUDA uint8 tensor of >= {nb} bytes")
            data = out[:nb]
        w = cls(m, n, q, g, has_offset, data, fmt=fmt)
        w.struct = lutgemm_weight(m, n, q, g, int(has_offset), int(fmt), data.data_ptr())
        return w

    def nbytes(self) -> int:
        return self.data.numel()


def lutgemm_pack_bcq(planes: torch.Tensor, alpha: torch.Tensor, offset: torch.Tensor | None, n: int, g: int,
                     stream=None, out: torch.Tensor | None = None) -> PackedBCQ:
    """Canonical BCQ (device tensors: planes int32/uint32 [q][m][n/32], alpha fp16
    [m][n/g][q], offset fp16 [m][n/g] or None) -> PackedBCQ (in `out`, a uint8 device view, if given)."""
    q, m = int(planes.shape[0]), int(planes.shape[1])
    for t in (planes, alpha, offset):
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("pack sources must be contiguous CUDA tensors")
    w = PackedBCQ.empty(m, n, q, g, offset is not None, planes.device, out=out)
    src = lutgemm_pack_src(SRC_BCQ, m, n, q, g, 0, planes.data_ptr(), alpha.data_ptr(), _ptr(offset), None, None,
                           None)
    _check("lutgemm_pack_bcq", lib.lutgemm_pack_bcq(ctypes.byref(src), ctypes.byref(w.struct), _stream(stream)))
    return w


def lutgemm_pack_uniform(codes: torch.Tensor, scale: torch.Tensor, zero: torch.Tensor, q: int, g: int,
                         stream=None, compact: bool = False) -> PackedBCQ:
    """Uniform codes (uint8 [m][n]), s and z_hat (fp16 [m][n/g]) -> extended BCQ (App. C).
    compact=True keeps one scale s per group (format UNIFORM_COMPACT, alpha_i derived in-kernel)."""
    m, n = int(codes.shape[0]), int(codes.shape[1])
    for t in (codes, scale, zero):
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("pack sources must be contiguous CUDA tensors")
    fmt = FMT_UNIFORM_COMPACT if compact else FMT_BCQ
    w = PackedBCQ.empty(m, n, q, g, True, codes.device, fmt)
    src = lutgemm_pack_src(SRC_UNIFORM_COMPACT if compact else SRC_UNIFORM, m, n, q, g, 0, None, None, None,
                           codes.data_ptr(), scale.data_ptr(), zero.data_ptr())
    _check("lutgemm_pack_bcq", lib.lutgemm_pack_bcq(ctypes.byref(src), ctypes.byref(w.struct), _stream(stream)))
    return w


def lutgemm_unpack_bcq(w: PackedBCQ, stream=None):
    """Native -> canonical (planes int32 [q][m][n/32], alpha fp16 [m][G][q], offset fp16 [m][G] | None)."""
    dev = w.data.device
    G = w.n // w.g  # g divides n
    planes = torch.empty((w.q, w.m, (w.n + 31) // 32), dtype=torch.int32, device=dev)
    alpha = torch.empty((w.m, G, w.q), dtype=torch.float16, device=dev)
    offset = torch.empty((w.m, G), dtype=torch.float16, device=dev) if w.has_offset else None
    _check("lutgemm_unpack_bcq", lib.lutgemm_unpack_bcq(ctypes.byref(w.struct), planes.data_ptr(), alpha.data_ptr(),
                                                        _ptr(offset), _stream(stream)))
    return planes, alpha, offset


def lutgemm_workspace_bytes(m: int, n: int, b: int = 1) -> int:
    return int(lib.lutgemm_workspace_bytes(m, n, b))


def make_workspace(nbytes: int, device, stream=None) -> torch.Tensor:
    ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
    _check("lutgemm_workspace_init", lib.lutgemm_workspace_init(ws.data_ptr(), ws.numel(), _stream(stream)))
    return ws


def lutgemm_gemv(w: PackedBCQ, x: torch.Tensor, y: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    """y[m] (fp16) = W x[n] (fp16)."""
    if y is None:
        y = torch.empty(w.m, dtype=torch.float16, device=x.device)
    if ws is None:
        ws = make_workspace(lutgemm_workspace_bytes(w.m, w.n, 1), x.device, stream)
    _check("lutgemm_gemv", lib.lutgemm_gemv(ctypes.byref(w.struct), x.data_ptr(), y.data_ptr(), ws.data_ptr(),
                                            ws.numel(), _stream(stream)))
    return y


def lutgemm_gemm_batched(w: PackedBCQ, X: torch.Tensor, Y: torch.Tensor | None = None,
                         ws: torch.Tensor | None = None, stream=None, f32: bool = False) -> torch.Tensor:
    """Y[b][m] = X[b][n] W^T, 1 <= b <= 32 (fp16 out, or fp32 with f32=True)."""
    b = int(X.shape[0])
    if Y is None:
        Y = torch.empty((b, w.m), dtype=torch.float32 if f32 else torch.float16, device=X.device)
    if ws is None:
        ws = make_workspace(lutgemm_workspace_bytes(w.m, w.n, b), X.device, stream)
    fn = lib.lutgemm_gemm_batched_f32 if f32 else lib.lutgemm_gemm_batched
    _check("lutgemm_gemm_batched", fn(ctypes.byref(w.struct), X.data_ptr(), b, Y.data_ptr(), ws.data_ptr(),
                                      ws.numel(), _stream(stream)))
    return Y


def lutgemm_host_workspace_bytes(m: int, n: int, b: int = 1) -> int:
    return int(lib.lutgemm_host_workspace_bytes(m, n, b))


def lutgemm_gemm_host(w: PackedBCQ, X_host: torch.Tensor, Y_host: torch.Tensor, ws: torch.Tensor, stream=None):
    """End-to-end: host X [b][n] -> device -> LUT-GEMM -> host Y [b][m] (synchronous)."""
    b = int(X_host.shape[0]) if X_host.dim() == 2 else 1
    _check("lutgemm_gemm_host", lib.lutgemm_gemm_host(ctypes.byref(w.struct), X_host.data_ptr(), b, Y_host.data_ptr(),
                                                      ws.data_ptr(), ws.numel(), _stream(stream)))
    return Y_host


def lutgemm_trace_enable(on: bool = True):
    _check("lutgemm_trace_enable", lib.lutgemm_trace_enable(int(on)))


def lutgemm_trace_read(ctas: int = 148):
    """Per-CTA timeline of the last traced launch: uint64 [ctas][8] (see lutgemm.h)."""
    import numpy as np
    buf = (ctypes.c_uint64 * (8 * ctas))()
    n = lib.lutgemm_trace_read(buf, 8 * ctas)
    return np.frombuffer(buf, dtype=np.uint64, count=n).reshape(-1, 8).copy()


# ---------------------------------------------------------------------------
# tensor parallelism
# ---------------------------------------------------------------------------

class TPComm:
    """NCCL communicator for lutgemm_tp_linear; the unique id travels over the
    caller's torch.distributed process group (plumbing only)."""

    def __init__(self, rank: int, world: int, group=None, device=None):
        import torch.distributed as dist
        idbuf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _check("lutgemm_tp_unique_id", lib.lutgemm_tp_unique_id(ctypes.cast(idbuf, _P)))
        backend = dist.get_backend(group)
        dev = device if (backend == "nccl") else "cpu"
        t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=0, group=group)
        raw = bytes(t.cpu().tolist())
        ctypes.memmove(idbuf, raw, 128)
        h = _P()
        _check("lutgemm_tp_init", lib.lutgemm_tp_init(world, rank, ctypes.cast(idbuf, _P), ctypes.byref(h)))
        self.handle = h
        self.rank, self.world = rank, world

    def workspace_bytes(self, mode: int, m_shard: int, n_shard: int, b: int) -> int:
        return int(lib.lutgemm_tp_workspace_bytes(self.handle, mode, m_shard, n_shard, b))

    def linear(self, mode: int, shard: PackedBCQ, x: torch.Tensor, y: torch.Tensor, ws: torch.Tensor, stream=None):
        b = int(x.shape[0]) if x.dim() == 2 else 1
        _check("lutgemm_tp_linear", lib.lutgemm_tp_linear(self.handle, mode, ctypes.byref(shard.struct), x.data_ptr(),
                                                          b, y.data_ptr(), ws.data_ptr(), ws.numel(),
                                                          _stream(stream)))
        return y

    def check(self):
        """Raise LutgemmError if the communicator hit an asynchronous NCCL error."""
        _check("lutgemm_tp_async_error", lib.lutgemm_tp_async_error(self.handle))

    def wait(self, stream=None, timeout_s: float = 300.0, poll_s: float = 0.001):
        """Wait for `stream` while polling the communicator for asynchronous errors (failure
        detection): on an NCCL error or after timeout_s the communicator is aborted (which
        releases kernels stuck in its collectives) and LutgemmError / TimeoutError is raised."""
        import time
        s = torch.cuda.current_stream() if stream is None else stream
        t0 = time.monotonic()
        while not s.query():
            st = lib.lutgemm_tp_async_error(self.handle)
            if st != OK:
                msg = lib.lutgemm_last_error().decode(errors="replace")
                self.abort()
                raise LutgemmError("lutgemm_tp_async_error", st, msg)
            if time.monotonic() - t0 > timeout_s:
                self.abort()
                raise TimeoutError(f"stream not done after {timeout_s} s; NCCL communicator aborted")
            time.sleep(poll_s)

    def abort(self):
        if self.handle:
            lib.lutgemm_tp_abort(self.handle)
            self.handle = None

    def close(self):
        if self.handle:
            _check("lutgemm_tp_destroy", lib.lutgemm_tp_destroy(self.handle))
            self.handle = None


def lutgemm_launch_count() -> int:
    """Product kernels launched by this process through the library (host-side count)."""
    return int(lib.lutgemm_launch_count())


def lutgemm_quantize_rtn(W: torch.Tensor, q: int, g: int, stream=None):
    """Dense fp16 W [m][n] (CUDA) -> (codes uint8 [m][n], scale fp16 [m][n/g], zero fp16 [m][n/g]): RTN."""
    if W.dtype != torch.float16 or not W.is_cuda or not W.is_contiguous():
        raise ValueError("W must be a contiguous CUDA fp16 tensor")
    m, n = int(W.shape[0]), int(W.shape[1])
    codes = torch.empty((m, n), dtype=torch.uint8, device=W.device)
    scale = torch.empty((m, n // g), dtype=torch.float16, device=W.device)
    zero = torch.empty((m, n // g), dtype=torch.float16, device=W.device)
    _check("lutgemm_quantize_rtn", lib.lutgemm_quantize_rtn(W.data_ptr(), m, n, q, g, codes.data_ptr(),
                                                            scale.data_ptr(), zero.data_ptr(), _stream(stream)))
    return codes, scale, zero


def lutgemm_quantize_bcq(W: torch.Tensor, q: int, g: int, iters: int = 0, stream=None):
    """Dense fp16 W [m][n] (CUDA) -> (planes int32 [q][m][n/32], alpha fp16 [m][n/g][q]): greedy BCQ
    plus `iters` alternating rounds."""
    if W.dtype != torch.float16 or not W.is_cuda or not W.is_contiguous():
        raise ValueError("W must be a contiguous CUDA fp16 tensor")
    m, n = int(W.shape[0]), int(W.shape[1])
    planes = torch.empty((q, m, n // 32), dtype=torch.int32, device=W.device)
    alpha = torch.empty((m, n // g, q), dtype=torch.float16, device=W.device)
    _check("lutgemm_quantize_bcq", lib.lutgemm_quantize_bcq(W.data_ptr(), m, n, q, g, iters, planes.data_ptr(),
                                                            alpha.data_ptr(), _stream(stream)))
    return planes, alpha


def lutgemm_p2p_window_bytes(world: int, mode: int, m: int) -> int:
    """Bytes of one exchange window: mode TP_ROWS_ALLGATHER (m = gathered rows) or TP_COLS_ALLREDUCE (m = rows)."""
    return int(lib.lutgemm_p2p_window_bytes(world, mode, m))


class P2PGroup:
    """Tensor-parallel exchange fused into the GEMV over peer memory (lutgemm_p2p_*):
    rows all-gather and column reduce-scatter + all-gather.  The 256-byte IPC records travel over the
    caller's torch.distributed group (plumbing only; gloo or nccl); one process per GPU (or, for
    testing, per process on one GPU).  Calls are CUDA-graph capturable.  ``rows_out`` / ``cols_m``
    size the windows for the largest gathered output / column-split layer the group will serve."""

    def __init__(self, rank: int, world: int, rows_out: int = 0, cols_m: int = 0, group=None):
        import torch.distributed as dist
        nbytes = max(lutgemm_p2p_window_bytes(world, TP_ROWS_ALLGATHER, rows_out) if rows_out else 0,
                     lutgemm_p2p_window_bytes(world, TP_COLS_ALLREDUCE, cols_m) if cols_m else 0)
        if nbytes <= 0:
            raise ValueError("P2PGroup needs rows_out > 0 or cols_m > 0")
        rec = (ctypes.c_uint8 * 256)()
        h = _P()
        _check("lutgemm_p2p_create", lib.lutgemm_p2p_create(rank, world, nbytes, ctypes.byref(h),
                                                            ctypes.cast(rec, _P)))
        self.handle, self.rank, self.world = h, rank, world
        try:
            if world > 1:
                recs = [None] * world
                dist.all_gather_object(recs, bytes(rec), group=group)
            else:
                recs = [bytes(rec)]
            allrec = (ctypes.c_uint8 * (256 * world)).from_buffer_copy(b"".join(recs))
            _check("lutgemm_p2p_connect", lib.lutgemm_p2p_connect(self.handle, ctypes.cast(allrec, _P)))
        except BaseException:
            lib.lutgemm_p2p_destroy(self.handle)
            self.handle = None
            raise

    def gemv_allgather(self, shard: PackedBCQ, x: torch.Tensor, ws: torch.Tensor, y: torch.Tensor,
                       stream=None) -> torch.Tensor:
        """Rows split: y (CUDA fp16 [world * m_shard]) = every rank's shard rows times x."""
        _check("lutgemm_p2p_gemv_allgather",
               lib.lutgemm_p2p_gemv_allgather(self.handle, ctypes.byref(shard.struct), x.data_ptr(), ws.data_ptr(),
                                              ws.numel(), _stream(stream), y.data_ptr()))
        return y

    def gemv_allreduce(self, shard: PackedBCQ, x_local: torch.Tensor, ws: torch.Tensor, y: torch.Tensor,
                       stream=None) -> torch.Tensor:
        """Column split: y [m] fp16 = sum over ranks of shard_r x_r (fused reduce-scatter + all-gather)."""
        _check("lutgemm_p2p_gemv_allreduce",
               lib.lutgemm_p2p_gemv_allreduce(self.handle, ctypes.byref(shard.struct), x_local.data_ptr(),
                                              ws.data_ptr(), ws.numel(), _stream(stream), y.data_ptr()))
        return y

    def close(self):
        if self.handle:
            _check("lutgemm_p2p_destroy", lib.lutgemm_p2p_destroy(self.handle))
            self.handle = None
