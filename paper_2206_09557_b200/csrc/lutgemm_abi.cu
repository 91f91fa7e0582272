// lutgemm_abi.cu -- the extern "C" boundary declared in include/lutgemm.h:
// argument validation, status codes, thread-local error text, dispatch.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "layout.cuh"
#include "lutgemm.h"
#include "lutgemm_internal.h"

namespace {

thread_local char g_err[512] = "";

lutgemm_status fail(lutgemm_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

lutgemm_status cuda_fail(cudaError_t e, const char* what) {
  return fail(LUTGEMM_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

lutgemm_status check_shape(int m, int n, int q, int g) {
  if (m < 1) return fail(LUTGEMM_ERR_INVALID_ARG, "m=%d must be >= 1", m);
  // n % 8, g % 8, g | n (g == n: row-wise); mu = 8 chunks never straddle a group (R13)
  if (n < 8 || n % 8) return fail(LUTGEMM_ERR_INVALID_ARG, "n=%d must be a positive multiple of 8", n);
  if (q < 1 || q > 8) return fail(LUTGEMM_ERR_INVALID_ARG, "q=%d must be in [1, 8]", q);
  if (g < 8 || g % 8 || n % g)
    return fail(LUTGEMM_ERR_INVALID_ARG, "g=%d must be a positive multiple of 8 that divides n=%d", g, n);
  if ((long long)m * ((n + 31) / 32) >= (1LL << 40)) return fail(LUTGEMM_ERR_INVALID_ARG, "shape too large");
  return LUTGEMM_OK;
}

// the compact uniform format holds one scale per (row, 32-column lane) at most: its kernels scale a
// lane's whole word by one s, so a group must not split a lane (g % 32 == 0 or row-wise)
lutgemm_status check_compact(int n, int g) {
  if (lg::group_class(n, g) == lg::kGrpChunk)
    return fail(LUTGEMM_ERR_INVALID_ARG,
                "the uniform-compact format needs g %% 32 == 0 or g == n (g=%d); pack with LUTGEMM_SRC_UNIFORM", g);
  return LUTGEMM_OK;
}

int g_dev_ok[64];  // 0 unknown, 1 ok, 2 unsupported

lutgemm_status check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= 64) dev = 0;
  if (!g_dev_ok[dev]) {
    int major = 0, minor = 0;
    e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    g_dev_ok[dev] = (major == 10 && minor == 0) ? 1 : 2;
    if (g_dev_ok[dev] == 2)
      return fail(LUTGEMM_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a only", dev, major,
                  minor);
  }
  if (g_dev_ok[dev] == 2) return fail(LUTGEMM_ERR_UNSUPPORTED, "device %d is not sm_100", dev);
  return LUTGEMM_OK;
}

lutgemm_status check_weight(const lutgemm_weight* w) {
  if (!w) return fail(LUTGEMM_ERR_INVALID_ARG, "weight is NULL");
  lutgemm_status st = check_shape(w->m, w->n, w->q, w->g);
  if (st != LUTGEMM_OK) return st;
  if (!w->data) return fail(LUTGEMM_ERR_INVALID_ARG, "weight data is NULL");
  if (w->has_offset != 0 && w->has_offset != 1) return fail(LUTGEMM_ERR_INVALID_ARG, "has_offset must be 0 or 1");
  if (!aligned(w->data, 16)) return fail(LUTGEMM_ERR_MISALIGNED, "weight data must be 16-byte aligned");
  if (w->format != LUTGEMM_FMT_BCQ && w->format != LUTGEMM_FMT_UNIFORM_COMPACT)
    return fail(LUTGEMM_ERR_INVALID_ARG, "bad weight format %d", w->format);
  if (w->format == LUTGEMM_FMT_UNIFORM_COMPACT && !w->has_offset)
    return fail(LUTGEMM_ERR_INVALID_ARG, "the uniform-compact format carries an offset (has_offset = 1)");
  if (w->format == LUTGEMM_FMT_UNIFORM_COMPACT) return check_compact(w->n, w->g);
  return LUTGEMM_OK;
}

lg::Shape weight_shape(const lutgemm_weight* w) {
  return lg::make_shape(w->m, w->n, w->q, w->g, w->has_offset, w->format == LUTGEMM_FMT_UNIFORM_COMPACT);
}

lutgemm_status product(const lutgemm_weight* w, const uint16_t* X, int b, uint16_t* Y, float* Yf, void* ws,
                       size_t ws_bytes, void* stream) {
  lutgemm_status st = check_weight(w);
  if (st != LUTGEMM_OK) return st;
  if (b < 1 || b > 32) return fail(LUTGEMM_ERR_INVALID_ARG, "b=%d must be in [1, 32]", b);
  if (!X || (!Y && !Yf) || !ws) return fail(LUTGEMM_ERR_INVALID_ARG, "x, y and ws must be non-NULL");
  if (!aligned(X, 16)) return fail(LUTGEMM_ERR_MISALIGNED, "x must be 16-byte aligned");
  if (!aligned(ws, 16)) return fail(LUTGEMM_ERR_MISALIGNED, "ws must be 16-byte aligned");
  if (Y && !aligned(Y, 2)) return fail(LUTGEMM_ERR_MISALIGNED, "y must be 2-byte aligned");
  if (Yf && !aligned(Yf, 4)) return fail(LUTGEMM_ERR_MISALIGNED, "yf must be 4-byte aligned");
  const lg::Shape sh = weight_shape(w);
  const size_t need = lg::workspace_bytes(sh, b);
  if (ws_bytes < need) return fail(LUTGEMM_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
  st = check_device();
  if (st != LUTGEMM_OK) return st;
  cudaError_t e = lg::run_product(sh, w->data, X, b, Y, Yf, ws, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "LUT-GEMM kernel launch");
  return LUTGEMM_OK;
}

}  // namespace

#ifndef LUTGEMM_SOURCE_HASH
#define LUTGEMM_SOURCE_HASH "unhashed-build----------"
#endif
// marker + 24 hex digits: _build.py finds it in the binary to decide whether to recompile
static const char kSourceHash[] = "LUTGEMM_SRC_HASH:" LUTGEMM_SOURCE_HASH;

extern "C" {

int lutgemm_abi_version(void) { return LUTGEMM_ABI_VERSION; }

const char* lutgemm_source_hash(void) { return kSourceHash + 17; }

const char* lutgemm_last_error(void) { return g_err; }

lutgemm_status lutgemm_packed_bytes(int m, int n, int q, int g, int has_offset, size_t* bytes) {
  lutgemm_status st = check_shape(m, n, q, g);
  if (st != LUTGEMM_OK) return st;
  if (!bytes) return fail(LUTGEMM_ERR_INVALID_ARG, "bytes is NULL");
  *bytes = lg::packed_bytes(lg::make_shape(m, n, q, g, has_offset));
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_packed_bytes_fmt(int m, int n, int q, int g, int has_offset, int format, size_t* bytes) {
  lutgemm_status st = check_shape(m, n, q, g);
  if (st != LUTGEMM_OK) return st;
  if (!bytes) return fail(LUTGEMM_ERR_INVALID_ARG, "bytes is NULL");
  if (format != LUTGEMM_FMT_BCQ && format != LUTGEMM_FMT_UNIFORM_COMPACT)
    return fail(LUTGEMM_ERR_INVALID_ARG, "bad format %d", format);
  if (format == LUTGEMM_FMT_UNIFORM_COMPACT && (st = check_compact(n, g)) != LUTGEMM_OK) return st;
  *bytes = lg::packed_bytes(lg::make_shape(m, n, q, g, has_offset, format == LUTGEMM_FMT_UNIFORM_COMPACT));
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_pack_bcq(const lutgemm_pack_src* src, lutgemm_weight* dst, void* stream) {
  if (!src || !dst) return fail(LUTGEMM_ERR_INVALID_ARG, "src/dst is NULL");
  lutgemm_status st = check_shape(src->m, src->n, src->q, src->g);
  if (st != LUTGEMM_OK) return st;
  const bool compact = src->kind == LUTGEMM_SRC_UNIFORM_COMPACT;
  const bool uniform = src->kind == LUTGEMM_SRC_UNIFORM || compact;
  if (src->kind != LUTGEMM_SRC_BCQ && !uniform) return fail(LUTGEMM_ERR_INVALID_ARG, "bad src kind %d", src->kind);
  if (compact && (st = check_compact(src->n, src->g)) != LUTGEMM_OK) return st;
  if (uniform) {
    if (!src->codes || !src->scale || !src->zero)
      return fail(LUTGEMM_ERR_INVALID_ARG, "uniform source needs codes, scale and zero");
  } else if (!src->planes || !src->alpha) {
    return fail(LUTGEMM_ERR_INVALID_ARG, "BCQ source needs planes and alpha");
  }
  const int has_offset = uniform ? 1 : (src->offset != nullptr);
  if (!dst->data) return fail(LUTGEMM_ERR_INVALID_ARG, "destination buffer not set");
  if (!aligned(dst->data, 16)) return fail(LUTGEMM_ERR_MISALIGNED, "destination buffer must be 16-byte aligned");
  if ((src->planes && !aligned(src->planes, 4)) || (src->alpha && !aligned(src->alpha, 2)) ||
      (src->offset && !aligned(src->offset, 2)) || (src->scale && !aligned(src->scale, 2)) ||
      (src->zero && !aligned(src->zero, 2)))
    return fail(LUTGEMM_ERR_MISALIGNED, "source buffers must be element-aligned");
  st = check_device();
  if (st != LUTGEMM_OK) return st;
  const lg::Shape sh = lg::make_shape(src->m, src->n, src->q, src->g, has_offset, compact);
  cudaError_t e;
  if (uniform)
    e = lg::run_pack_uniform(sh, src->codes, src->scale, src->zero, dst->data, static_cast<cudaStream_t>(stream));
  else
    e = lg::run_pack_bcq(sh, src->planes, src->alpha, src->offset, dst->data, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "pack kernel launch");
  dst->m = src->m;
  dst->n = src->n;
  dst->q = src->q;
  dst->g = src->g;
  dst->has_offset = has_offset;
  dst->format = compact ? LUTGEMM_FMT_UNIFORM_COMPACT : LUTGEMM_FMT_BCQ;
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_unpack_bcq(const lutgemm_weight* w, uint32_t* planes, uint16_t* alpha, uint16_t* offset,
                                  void* stream) {
  lutgemm_status st = check_weight(w);
  if (st != LUTGEMM_OK) return st;
  if (offset && !w->has_offset) return fail(LUTGEMM_ERR_INVALID_ARG, "weight has no offset to unpack");
  st = check_device();
  if (st != LUTGEMM_OK) return st;
  const lg::Shape sh = weight_shape(w);
  cudaError_t e = lg::run_unpack(sh, w->data, planes, alpha, offset, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "unpack kernel launch");
  return LUTGEMM_OK;
}

size_t lutgemm_workspace_bytes(int m, int n, int b) {
  if (m < 1 || n < 8 || b < 1) return 0;
  const lg::Shape sh = lg::make_shape(m, n, 1, n, 0);
  return lg::workspace_bytes(sh, b);
}

lutgemm_status lutgemm_workspace_init(void* ws, size_t ws_bytes, void* stream) {
  if (!ws) return fail(LUTGEMM_ERR_INVALID_ARG, "ws is NULL");
  cudaError_t e = cudaMemsetAsync(ws, 0, ws_bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(ws)");
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_gemv(const lutgemm_weight* w, const uint16_t* x, uint16_t* y, void* ws, size_t ws_bytes,
                            void* stream) {
  if (!y) return fail(LUTGEMM_ERR_INVALID_ARG, "y is NULL");
  return product(w, x, 1, y, nullptr, ws, ws_bytes, stream);
}

lutgemm_status lutgemm_gemm_batched(const lutgemm_weight* w, const uint16_t* X, int b, uint16_t* Y, void* ws,
                                    size_t ws_bytes, void* stream) {
  if (!Y) return fail(LUTGEMM_ERR_INVALID_ARG, "Y is NULL");
  return product(w, X, b, Y, nullptr, ws, ws_bytes, stream);
}

lutgemm_status lutgemm_gemm_batched_f32(const lutgemm_weight* w, const uint16_t* X, int b, float* Yf, void* ws,
                                        size_t ws_bytes, void* stream) {
  if (!Yf) return fail(LUTGEMM_ERR_INVALID_ARG, "Yf is NULL");
  return product(w, X, b, nullptr, Yf, ws, ws_bytes, stream);
}

static size_t align256(size_t v) { return (v + 255) / 256 * 256; }

size_t lutgemm_host_workspace_bytes(int m, int n, int b) {
  const size_t base = lutgemm_workspace_bytes(m, n, b);
  if (!base) return 0;
  return align256(base) + align256((size_t)b * n * 2) + align256((size_t)b * m * 2);
}

lutgemm_status lutgemm_gemm_host(const lutgemm_weight* w, const uint16_t* X_host, int b, uint16_t* Y_host, void* ws,
                                 size_t ws_bytes, void* stream) {
  lutgemm_status st = check_weight(w);
  if (st != LUTGEMM_OK) return st;
  if (!X_host || !Y_host || !ws) return fail(LUTGEMM_ERR_INVALID_ARG, "X_host, Y_host and ws must be non-NULL");
  if (b < 1 || b > 32) return fail(LUTGEMM_ERR_INVALID_ARG, "b=%d must be in [1, 32]", b);
  const size_t need = lutgemm_host_workspace_bytes(w->m, w->n, b);
  if (ws_bytes < need) return fail(LUTGEMM_ERR_WORKSPACE, "host workspace %zu bytes < required %zu", ws_bytes, need);
  const size_t pws = align256(lutgemm_workspace_bytes(w->m, w->n, b));
  uint8_t* xd = static_cast<uint8_t*>(ws) + pws;
  uint8_t* yd = xd + align256((size_t)b * w->n * 2);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // Y_host in page-locked, device-mapped memory (cudaHostAlloc / torch pin_memory under UVA): the
  // product's epilogue stores y straight into it over the host link (coalesced warp stores), no
  // separate device-to-host copy to launch and wait for.  x keeps its copy: every CTA of a slice
  // reads the slice, so reading x over the link would move it J times.
  uint16_t* y_mapped = nullptr;
  {
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, Y_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer)
      y_mapped = static_cast<uint16_t*>(pa.devicePointer);
    else
      cudaGetLastError();  // clear a query error on ordinary pageable memory
  }
  cudaError_t e = cudaMemcpyAsync(xd, X_host, (size_t)b * w->n * 2, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync H2D");
  st = product(w, reinterpret_cast<uint16_t*>(xd), b, y_mapped ? y_mapped : reinterpret_cast<uint16_t*>(yd), nullptr,
               ws, pws, stream);
  if (st != LUTGEMM_OK) return st;
  if (!y_mapped) {
    e = cudaMemcpyAsync(Y_host, yd, (size_t)b * w->m * 2, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync D2H");
  }
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return LUTGEMM_OK;
}

uint64_t lutgemm_launch_count(void) { return lg::launch_count(); }

lutgemm_status lutgemm_quantize_rtn(const uint16_t* W, int m, int n, int q, int g, uint8_t* codes, uint16_t* scale,
                                    uint16_t* zero, void* stream) {
  lutgemm_status st = check_shape(m, n, q, g);
  if (st != LUTGEMM_OK) return st;
  if (n % 32 || g % 32)  // the quantizers work on whole 32-column words (one warp lane per column)
    return fail(LUTGEMM_ERR_INVALID_ARG, "the quantizers need n %% 32 == 0 and g %% 32 == 0 (n=%d, g=%d)", n, g);
  if (!W || !codes || !scale || !zero) return fail(LUTGEMM_ERR_INVALID_ARG, "W, codes, scale and zero must be non-NULL");
  if (!aligned(W, 2) || !aligned(scale, 2) || !aligned(zero, 2))
    return fail(LUTGEMM_ERR_MISALIGNED, "fp16 buffers must be 2-byte aligned");
  st = check_device();
  if (st != LUTGEMM_OK) return st;
  cudaError_t e = lg::run_quantize_rtn(W, m, n, q, g, codes, scale, zero, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "quantize_rtn kernel launch");
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_quantize_bcq(const uint16_t* W, int m, int n, int q, int g, int iters, uint32_t* planes,
                                    uint16_t* alpha, void* stream) {
  lutgemm_status st = check_shape(m, n, q, g);
  if (st != LUTGEMM_OK) return st;
  if (n % 32 || g % 32)
    return fail(LUTGEMM_ERR_INVALID_ARG, "the quantizers need n %% 32 == 0 and g %% 32 == 0 (n=%d, g=%d)", n, g);
  if (iters < 0 || iters > 1000) return fail(LUTGEMM_ERR_INVALID_ARG, "iters=%d must be in [0, 1000]", iters);
  if (!W || !planes || !alpha) return fail(LUTGEMM_ERR_INVALID_ARG, "W, planes and alpha must be non-NULL");
  if (!aligned(W, 2) || !aligned(planes, 4) || !aligned(alpha, 2))
    return fail(LUTGEMM_ERR_MISALIGNED, "buffers must be element-aligned");
  if (lg::quantize_bcq_smem_per_warp(q, g) > 227u * 1024u)
    return fail(LUTGEMM_ERR_INVALID_ARG, "group of %d columns with q=%d exceeds the per-warp shared memory", g, q);
  st = check_device();
  if (st != LUTGEMM_OK) return st;
  cudaError_t e = lg::run_quantize_bcq(W, m, n, q, g, iters, planes, alpha, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "quantize_bcq kernel launch");
  return LUTGEMM_OK;
}

lutgemm_status lutgemm_trace_enable(int on) {
  lg::trace_enable(on);
  return LUTGEMM_OK;
}

size_t lutgemm_trace_read(uint64_t* host, size_t n) {
  return lg::trace_read(reinterpret_cast<unsigned long long*>(host), n);
}

}  // extern "C"

// exported for the TP / P2P translation units
lutgemm_status lutgemm_internal_fail(lutgemm_status st, const char* msg) { return fail(st, "%s", msg); }
lutgemm_status lutgemm_internal_check_weight(const lutgemm_weight* w) { return check_weight(w); }
lutgemm_status lutgemm_internal_check_device() { return check_device(); }
