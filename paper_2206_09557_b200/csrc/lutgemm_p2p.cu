// lutgemm_p2p.cu -- the rows all-gather of a tensor-parallel GEMV fused into the
// GEMV's epilogue over peer memory (the paper names the
// GPU-to-GPU communication as what limits tensor parallelism once the matmul is
// fast, Table 2).
//
// Every rank owns two output buffers (double buffer) and a signal counter,
// allocated with cudaMalloc and shared with the other ranks through CUDA IPC
// handles that the caller exchanges (any transport: the Python binding uses
// torch.distributed).  A call runs the fused GEMV whose reducer CTAs store each
// finished row of this rank's shard straight into buffer (round & 1) of every
// rank (NVLink / NVSwitch P2P stores), then the grid's last reducer signals
// every rank (red.release.sys) and then holds the grid open until this rank has
// received the round's P signals (ld.acquire.sys), so the kernel's completion
// means "gathered output ready" for whatever the stream runs next.  Flow control: a rank
// writes buffer (k+2) & 1 only after its wait for round k+1, which needs every
// peer's round-(k+1) signal, sent after that peer's stream ran everything before
// its round-(k+1) call -- including its consumers of round k.  Contract: the
// output of a call stays valid until the call after next; calls are made in the
// same order on every rank.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <new>

#include "layout.cuh"
#include "lutgemm.h"
#include "lutgemm_internal.h"

lutgemm_status lutgemm_internal_fail(lutgemm_status st, const char* msg);

struct lutgemm_p2p {
  int rank, nranks, dev;
  size_t out_bytes;
  void* out[2];          // local outputs
  unsigned* sig;         // local signal counter (256-byte block)
  void* peer_out[2][8];  // every rank's outputs in this process's address space (self: local)
  unsigned* peer_sig[8];
  bool connected;
  unsigned long long round;
};

namespace {

constexpr int kRec = 256;  // record: 3 IPC handles (64 B each), rank, out_bytes

lutgemm_status cuda_fail(cudaError_t e, const char* what) {
  char buf[384];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  return lutgemm_internal_fail(LUTGEMM_ERR_CUDA, buf);
}

}  // namespace

extern "C" {

lutgemm_status lutgemm_p2p_create(int rank, int nranks, size_t out_bytes, lutgemm_p2p** out, uint8_t record[256]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (!out || !record || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks || out_bytes == 0)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "bad p2p_create arguments (1 <= nranks <= 8)");
  lutgemm_p2p* g = new (std::nothrow) lutgemm_p2p;
  if (!g) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "out of host memory");
  memset(g, 0, sizeof(*g));
  g->rank = rank;
  g->nranks = nranks;
  g->out_bytes = (out_bytes + 255) / 256 * 256;
  cudaGetDevice(&g->dev);
  cudaError_t e = cudaMalloc(&g->out[0], g->out_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&g->out[1], g->out_bytes);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&g->sig), 256);
  if (e == cudaSuccess) e = cudaMemset(g->sig, 0, 256);
  memset(record, 0, kRec);
  cudaIpcMemHandle_t h[3];
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[0], g->out[0]);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[1], g->out[1]);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[2], g->sig);
  if (e != cudaSuccess) {
    lutgemm_p2p_destroy(g);
    return cuda_fail(e, "p2p buffers / IPC handles");
  }
  memcpy(record, h, 3 * 64);
  memcpy(record + 192, &rank, sizeof(int));
  const unsigned long long ob = g->out_bytes;
  memcpy(record + 200, &ob, sizeof(ob));
  *out = g;
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_p2p_connect(lutgemm_p2p* g, const uint8_t* records) {
  if (!g || !records) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "NULL argument");
  for (int pr = 0; pr < g->nranks; ++pr) {
    const uint8_t* rec = records + (size_t)pr * kRec;
    int r;
    unsigned long long ob;
    memcpy(&r, rec + 192, sizeof(int));
    memcpy(&ob, rec + 200, sizeof(ob));
    if (r != pr || ob != g->out_bytes)
      return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "records must be in rank order with equal out_bytes");
    if (pr == g->rank) {
      g->peer_out[0][pr] = g->out[0];
      g->peer_out[1][pr] = g->out[1];
      g->peer_sig[pr] = g->sig;
      continue;
    }
    cudaIpcMemHandle_t h[3];
    memcpy(h, rec, 3 * 64);
    void* p[3] = {nullptr, nullptr, nullptr};
    for (int i = 0; i < 3; ++i) {
      cudaError_t e = cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    }
    g->peer_out[0][pr] = p[0];
    g->peer_out[1][pr] = p[1];
    g->peer_sig[pr] = static_cast<unsigned*>(p[2]);
  }
  g->connected = true;
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_p2p_gemv_allgather(lutgemm_p2p* g, const lutgemm_weight* shard, const uint16_t* x, void* ws,
                                          size_t ws_bytes, void* stream, uint16_t** y_full, uint16_t* y_copy) {
  if (!g || !g->connected || !shard || !shard->data || !x || !ws)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "NULL argument or group not connected");
  const size_t m_total = (size_t)g->nranks * shard->m;
  if (m_total * 2 > g->out_bytes)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "output buffers too small for nranks * m_shard rows");
  if (lutgemm_workspace_bytes(shard->m, shard->n, 1) > ws_bytes)
    return lutgemm_internal_fail(LUTGEMM_ERR_WORKSPACE, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(ws) & 15) ||
      (reinterpret_cast<uintptr_t>(shard->data) & 15))
    return lutgemm_internal_fail(LUTGEMM_ERR_MISALIGNED, "x, ws and the weight must be 16-byte aligned");
  const lg::Shape sh = lg::make_shape(shard->m, shard->n, shard->q, shard->g, shard->has_offset,
                                      shard->format == LUTGEMM_FMT_UNIFORM_COMPACT);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int parity = (int)(g->round & 1);
  __half* peer_y[8];
  for (int pr = 0; pr < g->nranks; ++pr) peer_y[pr] = static_cast<__half*>(g->peer_out[parity][pr]);
  // the grid's last reducer waits for the round's P signals itself (no wait kernel)
  const unsigned target = (unsigned)((g->round + 1) * g->nranks);
  cudaError_t e = lg::run_gemv_p2p(sh, shard->data, x, ws, peer_y, g->peer_sig, g->nranks, g->rank * shard->m,
                                   g->rank, target, 0, st);
  if (e == cudaErrorNotSupported)
    return lutgemm_internal_fail(LUTGEMM_ERR_UNSUPPORTED, "shard shape does not run the fused GEMV mode");
  if (e != cudaSuccess) return cuda_fail(e, "fused GEMV launch");
  g->round += 1;
  if (y_copy) {
    e = cudaMemcpyAsync(y_copy, g->out[parity], m_total * 2, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "output copy");
  }
  if (y_full) *y_full = static_cast<uint16_t*>(g->out[parity]);
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_p2p_gemv_allreduce(lutgemm_p2p* g, const lutgemm_weight* shard, const uint16_t* x, void* ws,
                                          size_t ws_bytes, void* stream, uint16_t* y) {
  if (!g || !g->connected || !shard || !shard->data || !x || !ws || !y)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "NULL argument or group not connected");
  const size_t m = (size_t)shard->m;
  if ((size_t)g->nranks * m * 4 > g->out_bytes)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "buffers too small for nranks * m fp32 partial rows");
  if (lutgemm_workspace_bytes(shard->m, shard->n, 1) > ws_bytes)
    return lutgemm_internal_fail(LUTGEMM_ERR_WORKSPACE, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(ws) & 15) ||
      (reinterpret_cast<uintptr_t>(shard->data) & 15) || (reinterpret_cast<uintptr_t>(y) & 1))
    return lutgemm_internal_fail(LUTGEMM_ERR_MISALIGNED, "x, ws and the weight must be 16-byte aligned");
  const lg::Shape sh = lg::make_shape(shard->m, shard->n, shard->q, shard->g, shard->has_offset,
                                      shard->format == LUTGEMM_FMT_UNIFORM_COMPACT);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int parity = (int)(g->round & 1);
  __half* peer_y[8];
  for (int pr = 0; pr < g->nranks; ++pr) peer_y[pr] = static_cast<__half*>(g->peer_out[parity][pr]);
  const unsigned target = (unsigned)((g->round + 1) * g->nranks);
  // fp32 partial row r of this rank -> slot [rank][r] of every rank
  cudaError_t e = lg::run_gemv_p2p(sh, shard->data, x, ws, peer_y, g->peer_sig, g->nranks,
                                   (int)(g->rank * m), g->rank, target, 1, st);
  if (e == cudaErrorNotSupported)
    return lutgemm_internal_fail(LUTGEMM_ERR_UNSUPPORTED, "shard shape does not run the fused GEMV mode");
  if (e != cudaSuccess) return cuda_fail(e, "fused GEMV launch");
  g->round += 1;
  e = lg::launch_p2p_sum(static_cast<const float*>(g->out[parity]), g->nranks, (int)m, y, st);
  if (e != cudaSuccess) return cuda_fail(e, "p2p sum launch");
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_p2p_destroy(lutgemm_p2p* g) {
  if (!g) return LUTGEMM_OK;
  cudaDeviceSynchronize();
  for (int pr = 0; pr < g->nranks; ++pr) {
    if (pr == g->rank || !g->connected) continue;
    if (g->peer_out[0][pr]) cudaIpcCloseMemHandle(g->peer_out[0][pr]);
    if (g->peer_out[1][pr]) cudaIpcCloseMemHandle(g->peer_out[1][pr]);
    if (g->peer_sig[pr]) cudaIpcCloseMemHandle(g->peer_sig[pr]);
  }
  if (g->out[0]) cudaFree(g->out[0]);
  if (g->out[1]) cudaFree(g->out[1]);
  if (g->sig) cudaFree(g->sig);
  delete g;
  return LUTGEMM_OK;
}

}  // extern "C"
