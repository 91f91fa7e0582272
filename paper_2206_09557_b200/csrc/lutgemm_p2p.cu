// lutgemm_p2p.cu -- the tensor-parallel exchange of a LUT-GEMV fused into the GEMV's epilogue
// over peer memory (the paper names GPU-to-GPU communication as what limits
// tensor parallelism once the matmul is fast, Table 2).
//
// Every rank owns two exchange windows (double buffer, selected by the parity of a device-side
// round counter) allocated with cudaMalloc and shared through CUDA IPC handles that the caller
// exchanges (any transport; the Python binding uses torch.distributed).  A call is one kernel
// launch, graph-capturable (no host-side state changes between calls).
//
// The whole exchange runs in the fused GEMV's epilogue (gemv_kernel.cuh, p2p_epilogue), in the
// reducer CTAs, one thread per output row, as LL words over the NVLink / NVSwitch P2P mappings:
// 8-byte stores of 4 data bytes + a 4-byte round stamp, read back by polling the stamp (NCCL's
// LL protocol for small messages: no fence, no separate signal, no barrier).  Every rank runs
// the same reducer partition, so reducer (group, share) waits only for the same share's words
// of the other ranks:
//   rows (m-split, ROWS_ALLGATHER): fp16 row pairs of this rank's shard -> y and every peer's
//     window; the peers' rows of the same share out of the local window -> y;
//   cols (n-split, COLS_ALLREDUCE): reduce-scatter + all-gather: fp32 rows -> the row's OWNER
//     rank only (rank o owns rows [o mb, (o+1) mb)), slot [this rank]; the owner sums its rows
//     over the P slots in rank order (deterministic, identical on every rank), rounds to fp16 and
//     sends the row pairs to every peer; the other owners' rows out of the local window -> y.
// The last reducer advances the round.
//
// Flow control: window (k & 1) is rewritten in round k + 2 only; a rank enters round k + 2 after
// completing round k + 1, in which it received at least one round-(k+1) word from every peer
// (rows: every share reads every peer; columns: every rank owns rows, host-checked, and the
// owner reads every peer's slot), each written after that peer's stream completed its round-k
// call (round k + 1's epilogue starts after its PDL wait).  A stale word of the same parity
// carries stamp - 2; stamps are 32 bits, so a word would have to sit unwritten for a multiple
// of 2^32 rounds to be mistaken.  Every rank makes the same sequence of calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>

#include "kernels_common.cuh"
#include "lutgemm.h"

lutgemm_status lutgemm_internal_fail(lutgemm_status st, const char* msg);
lutgemm_status lutgemm_internal_check_weight(const lutgemm_weight* w);
lutgemm_status lutgemm_internal_check_device();

// signal block (device, 256 bytes): word 0 = the round (local; the LL words carry the signals)
constexpr int kRound = 0;
constexpr size_t kSigBytes = 256;

struct lutgemm_p2p {
  int rank, nranks, dev;
  size_t win_bytes;
  uint8_t* win[2];                     // local windows
  unsigned long long* sig;             // local signal block
  uint8_t* peer_win[2][8];             // every rank's windows in this process's address space (self: local)
  bool connected;
};

namespace {

using namespace lg;

constexpr int kRec = 256;  // record: 2 IPC handles (the windows, 64 B each), 64 B unused, rank, window bytes

lutgemm_status cuda_fail(cudaError_t e, const char* what) {
  char buf[384];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  return lutgemm_internal_fail(LUTGEMM_ERR_CUDA, buf);
}

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

// rows owned per rank in the column split (multiple of 8: 16-byte stores, whole 8-row units)
int block_rows(int m, int P) { return ((m + P - 1) / P + 7) / 8 * 8; }

lutgemm_status run(lutgemm_p2p* g, int mode, const lutgemm_weight* shard, const uint16_t* x, void* ws,
                   size_t ws_bytes, void* stream, uint16_t* y) {
  lutgemm_status st = lutgemm_internal_check_weight(shard);  // the shard first: shape errors name the shape
  if (st != LUTGEMM_OK) return st;
  if (!g || !g->connected || !x || !ws || !y)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "NULL argument or group not connected");
  const int P = g->nranks, ms = shard->m;
  if (mode == 1 && ms % 8)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "rows all-gather needs m_shard % 8 == 0");
  const int m_out = mode == 1 ? P * ms : ms;
  const int mb = block_rows(ms, P);
  if (mode == 2 && (long long)(P - 1) * mb >= ms)  // flow control needs a flag from every peer per call
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "column all-reduce: every rank must own rows (m too small for P)");
  const size_t need = lutgemm_p2p_window_bytes(P, mode == 1 ? LUTGEMM_TP_ROWS_ALLGATHER : LUTGEMM_TP_COLS_ALLREDUCE,
                                               m_out);
  if (need > g->win_bytes)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "exchange windows too small (lutgemm_p2p_window_bytes)");
  if (lutgemm_workspace_bytes(shard->m, shard->n, 1) > ws_bytes)
    return lutgemm_internal_fail(LUTGEMM_ERR_WORKSPACE, "workspace too small");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(ws) & 15) ||
      (reinterpret_cast<uintptr_t>(y) & 1))
    return lutgemm_internal_fail(LUTGEMM_ERR_MISALIGNED, "x and ws must be 16-byte aligned, y 2-byte aligned");
  st = lutgemm_internal_check_device();
  if (st != LUTGEMM_OK) return st;
  const lg::Shape sh = lg::make_shape(shard->m, shard->n, shard->q, shard->g, shard->has_offset,
                                      shard->format == LUTGEMM_FMT_UNIFORM_COMPACT);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  lg::P2PArgs a;
  for (int pr = 0; pr < 8; ++pr) {
    a.win[0][pr] = pr < P ? g->peer_win[0][pr] : nullptr;
    a.win[1][pr] = pr < P ? g->peer_win[1][pr] : nullptr;
  }
  a.round = g->sig + kRound;
  a.mode = mode;
  a.npeers = P;
  a.self = g->rank;
  a.yoff = mode == 1 ? g->rank * ms : 0;
  a.mb = mb;
  a.yarea = mode == 1 ? 0u : (unsigned)align256((size_t)P * mb * 8);
  cudaError_t e = lg::run_gemv_p2p(sh, shard->data, x, ws, a, y, s);
  if (e == cudaErrorNotSupported)
    return lutgemm_internal_fail(LUTGEMM_ERR_UNSUPPORTED, "shard shape does not run the fused GEMV mode");
  if (e != cudaSuccess) return cuda_fail(e, "fused GEMV launch");
  return LUTGEMM_OK;
}
}  // namespace

extern "C" {

size_t lutgemm_p2p_window_bytes(int nranks, int mode, int m) {
  if (nranks < 1 || nranks > 8 || m < 1) return 0;
  // LL words (8 bytes: 4 data + 4 stamp): rows = half2 per word; cols = fp32 slots, then half2 rows
  if (mode == LUTGEMM_TP_ROWS_ALLGATHER) return align256((size_t)m * 4);
  if (mode == LUTGEMM_TP_COLS_ALLREDUCE) {
    const size_t mb = (size_t)block_rows(m, nranks);
    return align256((size_t)nranks * mb * 8) + align256((size_t)nranks * mb * 4);
  }
  return 0;
}

lutgemm_status lutgemm_p2p_create(int rank, int nranks, size_t win_bytes, lutgemm_p2p** out, uint8_t record[256]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (!out || !record || nranks < 1 || nranks > 8 || rank < 0 || rank >= nranks || win_bytes == 0)
    return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "bad p2p_create arguments (1 <= nranks <= 8)");
  lutgemm_p2p* g = new (std::nothrow) lutgemm_p2p;
  if (!g) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "out of host memory");
  memset(g, 0, sizeof(*g));
  g->rank = rank;
  g->nranks = nranks;
  g->win_bytes = align256(win_bytes);
  cudaGetDevice(&g->dev);
  cudaError_t e = cudaMalloc(&g->win[0], g->win_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&g->win[1], g->win_bytes);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&g->sig), kSigBytes);
  if (e == cudaSuccess) e = cudaMemset(g->sig, 0, kSigBytes);
  if (e == cudaSuccess) e = cudaMemset(g->win[0], 0, g->win_bytes);
  if (e == cudaSuccess) e = cudaMemset(g->win[1], 0, g->win_bytes);
  memset(record, 0, kRec);
  cudaIpcMemHandle_t h[2];  // the windows (the signal block holds only the local round: not shared)
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[0], g->win[0]);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[1], g->win[1]);
  if (e != cudaSuccess) {
    lutgemm_p2p_destroy(g);
    return cuda_fail(e, "p2p windows / IPC handles");
  }
  memcpy(record, h, 2 * 64);
  memcpy(record + 192, &rank, sizeof(int));
  const unsigned long long wb = g->win_bytes;
  memcpy(record + 200, &wb, sizeof(wb));
  *out = g;
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_p2p_connect(lutgemm_p2p* g, const uint8_t* records) {
  if (!g || !records) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "NULL argument");
  if (g->connected) return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "group already connected");
  for (int pr = 0; pr < g->nranks; ++pr) {
    int r;
    unsigned long long wb;
    memcpy(&r, records + (size_t)pr * kRec + 192, sizeof(int));
    memcpy(&wb, records + (size_t)pr * kRec + 200, sizeof(wb));
    if (r != pr || wb != g->win_bytes)
      return lutgemm_internal_fail(LUTGEMM_ERR_INVALID_ARG, "records must be in rank order with equal window sizes");
  }
  for (int pr = 0; pr < g->nranks; ++pr) {
    if (pr == g->rank) {
      g->peer_win[0][pr] = g->win[0];
      g->peer_win[1][pr] = g->win[1];
      continue;
    }
    cudaIpcMemHandle_t h[2];
    memcpy(h, records + (size_t)pr * kRec, 2 * 64);
    void* p[2] = {nullptr, nullptr};
    for (int i = 0; i < 2; ++i) {
      cudaError_t e = cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        // close what this call opened (this peer's and every earlier peer's mappings)
        for (int j = 0; j < i; ++j) cudaIpcCloseMemHandle(p[j]);
        for (int q = 0; q < pr; ++q) {
          if (q == g->rank) continue;
          cudaIpcCloseMemHandle(g->peer_win[0][q]);
          cudaIpcCloseMemHandle(g->peer_win[1][q]);
          g->peer_win[0][q] = g->peer_win[1][q] = nullptr;
        }
        return cuda_fail(e, "cudaIpcOpenMemHandle");
      }
    }
    g->peer_win[0][pr] = static_cast<uint8_t*>(p[0]);
    g->peer_win[1][pr] = static_cast<uint8_t*>(p[1]);
  }
  g->connected = true;
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_p2p_gemv_allgather(lutgemm_p2p* g, const lutgemm_weight* shard, const uint16_t* x, void* ws,
                                          size_t ws_bytes, void* stream, uint16_t* y) {
  return run(g, 1, shard, x, ws, ws_bytes, stream, y);
}

lutgemm_status lutgemm_p2p_gemv_allreduce(lutgemm_p2p* g, const lutgemm_weight* shard, const uint16_t* x, void* ws,
                                          size_t ws_bytes, void* stream, uint16_t* y) {
  return run(g, 2, shard, x, ws, ws_bytes, stream, y);
}

lutgemm_status lutgemm_p2p_destroy(lutgemm_p2p* g) {
  if (!g) return LUTGEMM_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(g->dev);
  cudaDeviceSynchronize();
  for (int pr = 0; pr < g->nranks; ++pr) {
    if (pr == g->rank) continue;
    if (g->peer_win[0][pr]) cudaIpcCloseMemHandle(g->peer_win[0][pr]);
    if (g->peer_win[1][pr]) cudaIpcCloseMemHandle(g->peer_win[1][pr]);
  }
  if (g->win[0]) cudaFree(g->win[0]);
  if (g->win[1]) cudaFree(g->win[1]);
  if (g->sig) cudaFree(g->sig);
  cudaSetDevice(cur);
  delete g;
  return LUTGEMM_OK;
}

}  // extern "C"
