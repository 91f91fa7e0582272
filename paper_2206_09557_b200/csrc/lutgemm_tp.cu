// lutgemm_tp.cu -- tensor-parallel LUT-GEMM over NCCL (NVLink 5 / NVSwitch).
//
// The paper runs LUT-GEMM with model (tensor) parallelism on 1/2/4/8 GPUs
// (Table 2, Tables 3/4) and observes that the
// GPU-to-GPU communication becomes relatively larger once the matmul is fast
// (P:L411-413).  Two shardings:
//   * rows (m-split): local LUT-GEMM of rows [r m/P, (r+1) m/P); optional
//     ncclAllGather of the fp16 y slices -> bitwise equal to the 1-GPU rows;
//   * columns (n-split, multiple of g): local fp32 partial y over the local x
//     slice, ncclAllReduce(sum) in fp32, then one fp16 rounding.
// Everything is enqueued on the caller's stream, so the whole sequence is
// CUDA-graph capturable.  Links the NCCL that torch loads (pip 2.28.x).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <new>

#include "layout.cuh"
#include "lutgemm.h"
#include "lutgemm_internal.h"

lutgemm_status lutgemm_internal_fail(lutgemm_status st, const char* msg);

struct lutgemm_tp {
  ncclComm_t comm;
  int rank;
  int nranks;
};

namespace {

lutgemm_status nccl_fail(ncclResult_t r, const char* what) {
  char buf[384];
  snprintf(buf, sizeof(buf), "%s: %s", what, ncclGetErrorString(r));
  return lutgemm_internal_fail(LUTGEMM_ERR_NCCL, buf);
}

lutgemm_status cuda_fail(cudaError_t e, const char* what) {
  char buf[384];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  return lutgemm_internal_fail(LUTGEMM_ERR_CUDA, buf);
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

// extra buffers after the product workspace
size_t tp_extra_bytes(int P, int mode, int ms, int b) {
  if (mode == LUTGEMM_TP_ROWS_ALLGATHER && b > 1)
    return align256((size_t)b * ms * 2) + align256((size_t)P * b * ms * 2);
  if (mode == LUTGEMM_TP_COLS_ALLREDUCE) return align256((size_t)b * ms * 4);
  return 0;
}

}  // namespace

extern "C" {

lutgemm_status lutgemm_tp_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  if (!id) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "id is NULL");
  ncclUniqueId uid;
  ncclResult_t r = ncclGetUniqueId(&uid);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id, &uid, 128);
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_tp_init(int nranks, int rank, const uint8_t id[128], lutgemm_tp** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "bad tp_init arguments");
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  lutgemm_tp* tp = new (std::nothrow) lutgemm_tp;
  if (!tp) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "out of host memory");
  ncclResult_t r = ncclCommInitRank(&tp->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete tp;
    return nccl_fail(r, "ncclCommInitRank");
  }
  tp->rank = rank;
  tp->nranks = nranks;
  *out = tp;
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_tp_async_error(lutgemm_tp* tp) {
  if (!tp) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "tp is NULL");
  ncclResult_t async = ncclSuccess;
  ncclResult_t r = ncclCommGetAsyncError(tp->comm, &async);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
  if (async != ncclSuccess && async != ncclInProgress) return nccl_fail(async, "NCCL asynchronous error");
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_tp_abort(lutgemm_tp* tp) {
  if (!tp) return LUTGEMM_OK;
  ncclResult_t r = ncclCommAbort(tp->comm);
  delete tp;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommAbort");
  return LUTGEMM_OK;
}

int lutgemm_tp_rank(const lutgemm_tp* tp) { return tp ? tp->rank : -1; }
int lutgemm_tp_nranks(const lutgemm_tp* tp) { return tp ? tp->nranks : -1; }

size_t lutgemm_tp_workspace_bytes(const lutgemm_tp* tp, int mode, int m_shard, int n_shard, int b) {
  if (!tp || m_shard < 1 || n_shard < 32 || b < 1) return 0;
  return align256(lutgemm_workspace_bytes(m_shard, n_shard, b)) + tp_extra_bytes(tp->nranks, mode, m_shard, b);
}

lutgemm_status lutgemm_tp_linear(lutgemm_tp* tp, int mode, const lutgemm_weight* shard, const uint16_t* x, int b,
                                 uint16_t* y, void* ws, size_t ws_bytes, void* stream) {
  if (!tp || !shard || !y || !ws) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "NULL argument");
  if (mode < LUTGEMM_TP_ROWS_LOCAL || mode > LUTGEMM_TP_COLS_ALLREDUCE)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "bad TP mode");
  if (b < 1 || b > 32) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "b must be in [1, 32]");
  const int ms = shard->m;
  const size_t need = lutgemm_tp_workspace_bytes(tp, mode, ms, shard->n, b);
  if (ws_bytes < need) return lutgemm_internal_fail(LUTGEMM_ERR_WORKSPACE, "TP workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t pws = align256(lutgemm_workspace_bytes(ms, shard->n, b));
  uint8_t* extra = static_cast<uint8_t*>(ws) + pws;
  const int P = tp->nranks;
  lutgemm_status s;
  ncclResult_t r;
  switch (mode) {
    case LUTGEMM_TP_ROWS_LOCAL:
      return lutgemm_gemm_batched(shard, x, b, y, ws, pws, stream);
    case LUTGEMM_TP_ROWS_ALLGATHER:
      if (b == 1) {
        uint16_t* mine = y + (size_t)tp->rank * ms;
        s = lutgemm_gemv(shard, x, mine, ws, pws, stream);
        if (s != LUTGEMM_OK) return s;
        r = ncclAllGather(mine, y, (size_t)ms, ncclHalf, tp->comm, st);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
        return LUTGEMM_OK;
      } else {
        uint16_t* local = reinterpret_cast<uint16_t*>(extra);
        uint16_t* gath = reinterpret_cast<uint16_t*>(extra + align256((size_t)b * ms * 2));
        s = lutgemm_gemm_batched(shard, x, b, local, ws, pws, stream);
        if (s != LUTGEMM_OK) return s;
        r = ncclAllGather(local, gath, (size_t)b * ms, ncclHalf, tp->comm, st);
        if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
        cudaError_t e = lg::run_gather_permute(gath, y, P, b, ms, st);
        if (e != cudaSuccess) return cuda_fail(e, "gather permute");
        return LUTGEMM_OK;
      }
    case LUTGEMM_TP_COLS_ALLREDUCE: {
      float* yf = reinterpret_cast<float*>(extra);
      s = lutgemm_gemm_batched_f32(shard, x, b, yf, ws, pws, stream);
      if (s != LUTGEMM_OK) return s;
      r = ncclAllReduce(yf, yf, (size_t)b * ms, ncclFloat, ncclSum, tp->comm, st);
      if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
      cudaError_t e = lg::run_cast_f32_f16(yf, y, (size_t)b * ms, st);
      if (e != cudaSuccess) return cuda_fail(e, "cast");
      return LUTGEMM_OK;
    }
  }
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_tp_destroy(lutgemm_tp* tp) {
  if (!tp) return LUTGEMM_OK;
  ncclResult_t r = ncclCommDestroy(tp->comm);
  delete tp;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return LUTGEMM_OK;
}

}  // extern "C"
