"""B200-native LUT-GEMM (arXiv 2206.09557): the quantized GEMV/GEMM hot path.

The compute lives in ``liblutgemm.so`` (sm_100a CUDA kernels behind the C ABI
of ``include/lutgemm.h``); ``lutgemm`` is its ctypes binding.  Importing this
package without the built library raises -- there is no CPU fallback.
"""
from .lutgemm import (  # noqa: F401
    FMT_BCQ,
    FMT_UNIFORM_COMPACT,
    LIB_PATH,
    LutgemmError,
    P2PGroup,
    PackedBCQ,
    TPComm,
    TP_COLS_ALLREDUCE,
    TP_ROWS_ALLGATHER,
    TP_ROWS_LOCAL,
    lutgemm_gemm_batched,
    lutgemm_gemm_host,
    lutgemm_trace_enable,
    lutgemm_trace_read,
    lutgemm_gemv,
    lutgemm_host_workspace_bytes,
    lutgemm_launch_count,
    lutgemm_pack_bcq,
    lutgemm_pack_uniform,
    lutgemm_quantize_bcq,
    lutgemm_quantize_rtn,
    lutgemm_packed_bytes,
    lutgemm_unpack_bcq,
    lutgemm_workspace_bytes,
    make_workspace,
)
