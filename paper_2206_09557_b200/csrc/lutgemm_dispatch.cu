// lutgemm_dispatch.cu -- host side of the products: work planning (fused
// mode, reducers, batched split), workspace sizes, launch glue, tracing.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "kernels_common.cuh"

namespace lg {

static int g_num_sms[64];

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!g_num_sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms[dev] = v > 0 ? v : 148;
  }
  return g_num_sms[dev];
}

cudaError_t ensure_smem_attr(const void* kernel) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == kernel && d.second == dev) return cudaSuccess;
  // the attribute is what the launches request (not the 227 KB opt-in maximum): the shared-memory
  // carveout follows it, and every KB not taken from the L1 keeps load sectors in flight
  static const int smax = getenv("LUTGEMM_SMEM_ATTR") ? atoi(getenv("LUTGEMM_SMEM_ATTR")) : kSmemBytesBase;
  const cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
  if (err == cudaSuccess) done.emplace_back(kernel, dev);
  return err;
}

const cudaLaunchAttribute* pdl_attr() {
  static const cudaLaunchAttribute a = [] {
    cudaLaunchAttribute x;
    x.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    x.val.programmaticStreamSerializationAllowed = 1;
    return x;
  }();
  return &a;
}

std::atomic<unsigned long long> g_launches{0};

// arrival counters and epochs of the fused reduction, then the grid-wide
// done counter of the fused rows all-gather (256-byte aligned)
// [2][kFusedMaxJ] arrival / departure counters, 64 misc words (the P2P round-advance counter at word 2)
static size_t counters_bytes(const Shape&) { return 2u * kFusedMaxJ * 4u + 256u; }

int batch_pad(int b) {
  int bp = 1;
  while (bp < b) bp <<= 1;
  return b == 1 ? 1 : (b == 2 ? 2 : std::max(bp, 4));
}

size_t workspace_bytes(const Shape& sh, int b) {
  // b <= 4: sub-slice partials of the GEMV-structured kernel ([V S][b][m4], V = 2 or 4)
  const size_t slices = b == 2 ? 2 * (size_t)sh.S : (b <= 4 && b > 1 ? 4 * (size_t)sh.S : (size_t)sh.S);
  const size_t own = counters_bytes(sh) + (slices * (size_t)batch_pad(b) * (size_t)sh.m4 * 4u + 255) / 256 * 256;
  // b > 4 runs either the vector-slot kernel or (batch_split) chunks of <= 4 rows: room for both
  return b > 4 ? std::max(own, workspace_bytes(sh, 4)) : own;
}

// b > 4 (and b = 3) as chunks of 4, 2 and 1 activation rows through the GEMV-structured kernels
// instead of the vector-slot kernel (b > 4) or a padded V = 4 pass (b = 3): those run nearer their
// shared-memory roof (fc1: b = 1 / 2 / 3 / 4 in 47 / 79 / 140 / 143 us against b = 5..8 in 318 us
// in the vector-slot kernel, which pads to 8), and the re-read weights hide under the lookups.
// A remainder of 3 runs as 2 + 1.  Not for chunk-group shapes (g % 32 != 0), which only the
// vector-slot kernel serves.  LUTGEMM_BATCH_SPLIT=0 keeps the single launch (tests, sweeps).
static bool batch_split(const Shape& sh, int b) {
  static const int env = getenv("LUTGEMM_BATCH_SPLIT") ? atoi(getenv("LUTGEMM_BATCH_SPLIT")) : 1;
  static const int vslot = getenv("LUTGEMM_SMALLB_BATCHED") ? atoi(getenv("LUTGEMM_SMALLB_BATCHED")) : 0;
  return env && !vslot && (b > 4 || b == 3) && sh.gcls != kGrpChunk;
}

static unsigned long long* g_trace = nullptr;
static bool g_trace_on = false;
constexpr int kTraceMaxCtas = 1024;

unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

void trace_enable(int on) {
  g_trace_on = on != 0;
  if (g_trace_on && !g_trace) cudaMalloc(&g_trace, sizeof(unsigned long long) * kTraceSlots * kTraceMaxCtas);
  if (g_trace_on && g_trace) cudaMemset(g_trace, 0, sizeof(unsigned long long) * kTraceSlots * kTraceMaxCtas);
}

size_t trace_read(unsigned long long* host, size_t n) {
  if (!g_trace || !host) return 0;
  const size_t cap = (size_t)kTraceSlots * kTraceMaxCtas;
  if (n > cap) n = cap;
  cudaMemcpy(host, g_trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return n;
}

// fused mode of the GEMV-structured kernels: S slices x J CTAs with J = #SMs / S,
// idling at most 8 % of the SMs, and at least J row units per slice
static bool fusable(int S, int units, int sms) {
  const char* env = getenv("LUTGEMM_FUSE_MIN_PCT");  // tuning / tests (>100 disables the fused mode)
  const int min_pct = env ? atoi(env) : 80;
  const int J = S <= sms ? sms / S : 0;
  return J >= 1 && J <= kFusedMaxJ && S <= kFusedMaxJ && S * J * 100 >= sms * min_pct && units >= J &&
         (long long)units * J < (1LL << 31);  // the kernels' 32-bit row-group arithmetic
}

static cudaError_t run_product_ex(const Shape& sh, const void* data, const uint16_t* x, int b, uint16_t* y, float* yf,
                                  void* ws, cudaStream_t st, const P2PArgs* pa);

cudaError_t run_product(const Shape& sh, const void* data, const uint16_t* x, int b, uint16_t* y, float* yf,
                        void* ws, cudaStream_t st) {
  if (batch_split(sh, b)) {  // rows [c0, c0 + cb) of X and Y, one after the other on the stream
    for (int c0 = 0, cb; c0 < b; c0 += cb) {
      cb = b - c0 >= 4 ? 4 : (b - c0 == 3 ? 2 : b - c0);
      const cudaError_t e = run_product_ex(sh, data, x + (size_t)c0 * sh.n, cb, y ? y + (size_t)c0 * sh.m : nullptr,
                                           yf ? yf + (size_t)c0 * sh.m : nullptr, ws, st, nullptr);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  return run_product_ex(sh, data, x, b, y, yf, ws, st, nullptr);
}

cudaError_t run_gemv_p2p(const Shape& sh, const void* data, const uint16_t* x, void* ws, const P2PArgs& a,
                         uint16_t* y, cudaStream_t st) {
  if (a.npeers < 1 || a.npeers > 8 || a.self < 0 || a.self >= a.npeers || (a.mode != 1 && a.mode != 2))
    return cudaErrorInvalidValue;
  return run_product_ex(sh, data, x, 1, y, nullptr, ws, st, &a);
}

static cudaError_t run_product_ex(const Shape& sh, const void* data, const uint16_t* x, int b, uint16_t* y, float* yf,
                                  void* ws, cudaStream_t st, const P2PArgs* pa) {
  KParams p{};
  p.p2p_mode = pa ? pa->mode : 0;
  p.npeers = pa ? pa->npeers : 0;
  p.yoff = pa ? pa->yoff : 0;
  p.p2p_self = pa ? pa->self : 0;
  p.p2p_mb = pa ? pa->mb : 0;
  p.p2p_yarea = pa ? pa->yarea : 0;
  p.p2p_round = pa ? pa->round : nullptr;
  {
    static const long long tmo = getenv("LUTGEMM_P2P_TIMEOUT_MS") ? atoll(getenv("LUTGEMM_P2P_TIMEOUT_MS")) : 30000;
    p.p2p_timeout_ns = (unsigned long long)std::max(1LL, tmo) * 1000000ull;
  }
  for (int i = 0; i < 8; ++i) {
    const bool on = pa && i < pa->npeers;
    p.p2p_win[0][i] = on ? pa->win[0][i] : nullptr;
    p.p2p_win[1][i] = on ? pa->win[1][i] : nullptr;
  }
  p.data = static_cast<const uint8_t*>(data);
  p.x = reinterpret_cast<const __half*>(x);
  p.y = reinterpret_cast<__half*>(y);
  p.yf = yf;
  p.counters = static_cast<unsigned*>(ws);
  p.partial = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + counters_bytes(sh));
  p.sh = sh;
  p.fs = full_slice(sh);
  p.b = b;
  int bl = 0;
  while ((1 << bl) < batch_pad(b)) ++bl;
  p.bl = bl;
  p.nv = b == 2 ? 1 : (1 << bl) / 4;
  p.spi = 1;
  p.qpw = 256;
  {
    static unsigned seq = 0;  // consecutive launches alternate between two halves of the trace buffer
    p.trace = g_trace_on ? g_trace + (size_t)(seq++ & 1u) * (kTraceMaxCtas / 2) * kTraceSlots : nullptr;
  }
  const bool batched = b > 1;
  p.s2 = 0;
  if (!batched) {
    p.items = (long long)sh.S * sh.RQ;
  } else if (b <= 4 && sh.gcls != kGrpChunk &&
             !(getenv("LUTGEMM_SMALLB_BATCHED") && atoi(getenv("LUTGEMM_SMALLB_BATCHED")))) {
    // b <= 4: GEMV-structured kernel over sub-slices of 1024 / V columns, V = 2 (b = 2)
    // or 4 (b = 3, 4); LUTGEMM_SMALLB_BATCHED=1 selects the vector-slot batched kernel
    const int V = b == 2 ? 2 : 4;
    p.s2 = (sh.n + 1024 / V - 1) / (1024 / V);
    p.items = (long long)p.s2 * ((sh.RQ + V - 1) / V);
  } else {
    p.spi = 0;
    plan_batched(sh, num_sms(), p);
  }
  int grid = (int)std::min<long long>((long long)num_sms(), p.items);
  // fused mode (b = 1): whole slices per CTA group, S*J CTAs with J per slice,
  // when that idles at most 20 % of the SMs; the reduction then runs in-kernel
  // with R reducers per row-quad group (~16 KB of partials each; the others
  // exit early).  LUTGEMM_GEMV_REDUCERS overrides R (tests, tuning).
  p.fused_J = 0;
  p.reducers = 0;
  if (p.s2 > 0) {  // b <= 4 kernel: the GEMV's fused mode over sub-slices
    const int sms = num_sms();
    const int V = b == 2 ? 2 : 4;
    const int NG = (sh.RQ + V - 1) / V;
    const int J = p.s2 <= sms ? sms / p.s2 : 0;
    if (fusable(p.s2, NG, sms)) {
      p.fused_J = J;
      grid = p.s2 * J;
      for (int fj = 0; fj <= J; ++fj) p.gq[fj] = (int)((long long)NG * fj / J);
      p.rcp_J = 1.0f / (float)J;
      const long long red_bytes = (long long)p.s2 * b * 4 * (4 * V) * ((NG + J - 1) / J);
      p.reducers = (int)std::min<long long>(p.s2, (red_bytes + 16383) / 16384);
    }
  }
  p.smem_bytes = kSmemBytesBase;
  {
    static const int xd = getenv("LUTGEMM_XDIRECT") ? atoi(getenv("LUTGEMM_XDIRECT")) : 1;
    p.xdirect = xd;
  }
  if (!batched) {
    const int sms = num_sms();
    const int J = sh.S <= sms ? sms / sh.S : 0;
    if (fusable(sh.S, pa ? (sh.RQ + 1) / 2 : sh.RQ, sms)) {
      p.fused_J = J;
      grid = sh.S * J;
      // row-quad groups; with the P2P epilogue they start on even quads (its 8-row units)
      for (int fj = 0; fj <= J; ++fj)
        p.gq[fj] = !pa ? (int)((long long)sh.RQ * fj / J)
                       : std::min(sh.RQ, 2 * (int)((long long)((sh.RQ + 1) / 2) * fj / J));
      p.rcp_J = 1.0f / (float)J;
      const long long red_bytes = (long long)sh.S * 16 * ((sh.RQ + J - 1) / J);
      p.reducers = (int)std::min<long long>(sh.S, (red_bytes + 8191) / 8192);  // ~8 KB of partials per reducer
      const char* env = getenv("LUTGEMM_GEMV_REDUCERS");
      if (env && atoi(env) > 0) p.reducers = std::min(atoi(env), sh.S);
    }
  }
  if (pa && (batched || p.fused_J <= 0)) return cudaErrorNotSupported;  // the fused epilogue only
  cudaError_t e = !batched ? launch_gemv(p, grid, st) : (p.s2 > 0 ? launch_smallb(p, grid, st) : launch_batched(p, grid, st));
  if (e != cudaSuccess) return e;
  if (p.fused_J > 0) return cudaSuccess;  // reduced in-kernel
  if (p.s2 > 0) {  // sub-slice partials [SV][b][m4]: the GEMV reduction kernel with S = SV
    KParams r = p;
    r.sh.S = p.s2;
    return launch_reduce(r, st);
  }
  return batched ? launch_reduce_batched(p, st) : launch_reduce(p, st);
}

}  // namespace lg
