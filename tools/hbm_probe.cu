// hbm_probe.cu -- calibration micro-kernels for the LUT-GEMM roofline:
// achievable HBM read bandwidth with the access patterns the LUT kernel can use,
// and the conflict-free shared-memory lookup rate.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/hbm_probe tools/hbm_probe.cu && build/hbm_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint4 ldg_na(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Each CTA streams a contiguous chunk; warps take 512-byte rows round-robin,
// U loads in flight per thread, optional bulk L2 prefetch PF rows ahead per warp-step.
template <int U>
__global__ void __launch_bounds__(512) stream_ldg(const uint8_t* __restrict__ buf, size_t bytes, int pf_bytes,
                                                  uint32_t* out) {
  const size_t per = bytes / gridDim.x / 512 * 512;
  const uint8_t* base = buf + (size_t)blockIdx.x * per;
  const int nrow = (int)(per / 512);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint32_t acc = 0;
  if (pf_bytes > 0 && threadIdx.x == 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base), "r"((uint32_t)pf_bytes) : "memory");
  for (int r0 = warp; r0 < nrow; r0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * nw;
      v[u] = r < nrow ? ldg_na(base + (size_t)r * 512 + lane * 16) : make_uint4(0, 0, 0, 0);
    }
    if (pf_bytes > 0 && threadIdx.x == 0) {
      const size_t off = (size_t)(r0 + nw * U) * 512 + pf_bytes;
      if (off + nw * U * 512 <= per)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"((uint32_t)(nw * U * 512))
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// Ring-structured stream like the LUT kernel: each warp owns row quads
// rq = warp + 16 t of a contiguous per-CTA range; a quad is 3 x 512 bytes
// (3 planes); PD quads in flight per warp; between a quad's arrival and its
// reload the warp executes `work` dependent-free ALU ops per plane word.
template <int PD>
__global__ void __launch_bounds__(512, 1) ring_stream(const uint8_t* __restrict__ buf, size_t bytes, int work,
                                                     uint32_t* out) {
  const size_t per = bytes / gridDim.x / 1536 * 1536;
  const uint8_t* base = buf + (size_t)blockIdx.x * per;
  const int nq = (int)(per / 1536);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4 r[PD][3];
#pragma unroll
  for (int d = 0; d < PD; ++d) {
    const int rq = warp + 16 * d;
#pragma unroll
    for (int i = 0; i < 3; ++i) r[d][i] = rq < nq ? ldg_na(base + (size_t)rq * 1536 + i * 512 + lane * 16) : make_uint4(0,0,0,0);
  }
  uint32_t acc = 0;
  for (int rq0 = warp; rq0 < nq; rq0 += 16 * PD) {
#pragma unroll
    for (int d = 0; d < PD; ++d) {
      const int rq = rq0 + 16 * d;
      if (rq < nq) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          uint32_t a = r[d][i].x, b = r[d][i].y, c = r[d][i].z, e = r[d][i].w;
          for (int k = 0; k < work; ++k) {
            a = __byte_perm(a, b, 0x7604); b = __byte_perm(b, c, 0x7615);
            c = __byte_perm(c, e, 0x7624); e = __byte_perm(e, a, 0x7635);
          }
          acc ^= a ^ b ^ c ^ e;
        }
        const int rn = rq + 16 * PD;
#pragma unroll
        for (int i = 0; i < 3; ++i) r[d][i] = rn < nq ? ldg_na(base + (size_t)rn * 1536 + i * 512 + lane * 16) : make_uint4(0,0,0,0);
      }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// Batched structure: each warp loads U quads (3 x 512 B each) at once, then
// computes on them; DB = double-buffered (next batch requested before computing).
template <int U, bool DB, bool CONTIG>
__global__ void __launch_bounds__(512, 1) batch_stream(const uint8_t* __restrict__ buf, size_t bytes, int work,
                                                      uint32_t* out) {
  const size_t per = bytes / gridDim.x / 1536 * 1536;
  const uint8_t* base = buf + (size_t)blockIdx.x * per;
  const int nq = (int)(per / 1536);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CONTIG: warp w owns quads [w*nq/16, (w+1)*nq/16); else quads w + 16 t
  const int q0 = CONTIG ? warp * nq / 16 : warp, q1 = CONTIG ? (warp + 1) * nq / 16 : nq;
  const int qs = CONTIG ? 1 : 16;
  auto qidx = [&](int t) { return q0 + t * qs; };
  const int nt = CONTIG ? (q1 - q0) : (nq - warp + 15) / 16;
  uint4 cur[U][3], nxt[U][3];
  auto load = [&](uint4 (&r)[U][3], int t0) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + u;
#pragma unroll
      for (int i = 0; i < 3; ++i)
        r[u][i] = t < nt ? ldg_na(base + (size_t)qidx(t) * 1536 + i * 512 + lane * 16) : make_uint4(0, 0, 0, 0);
    }
  };
  uint32_t acc = 0;
  if (DB) load(nxt, 0);
  for (int t0 = 0; t0 < nt; t0 += U) {
    if (DB) {
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < 3; ++i) cur[u][i] = nxt[u][i];
      load(nxt, t0 + U);
    } else {
      load(cur, t0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        uint32_t a = cur[u][i].x, b = cur[u][i].y, c = cur[u][i].z, e = cur[u][i].w;
        for (int k = 0; k < work; ++k) {
          a = __byte_perm(a, b, 0x7604); b = __byte_perm(b, c, 0x7615);
          c = __byte_perm(c, e, 0x7624); e = __byte_perm(e, a, 0x7635);
        }
        acc ^= a ^ b ^ c ^ e;
      }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// Conflict-free random lookups: lane l reads table slot l (bank l) at a random key, like the LUT kernel.
__global__ void __launch_bounds__(512) lds_rate(int iters, uint32_t* out) {
  extern __shared__ float lut[];
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) lut[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t k = threadIdx.x * 2654435761u;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      k = k * 1664525u + 1013904223u;
      acc += lut[((k >> 24) << 6) + lane + ((u & 1) << 5)];
    }
  }
  if (acc == 1.2345f) out[0] = 1;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t bytes = (size_t)2 << 30;  // 2 GiB, far above L2
  uint8_t* buf;
  uint32_t* out;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&out, 64));
  CK(cudaMemset(buf, 1, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch, const char* name, double nbytes) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    const int R = 10;
    for (int i = 0; i < R; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-48s %8.1f GB/s  (%.1f us/launch)\n", name, nbytes * R / (ms * 1e-3) / 1e9, ms * 1e3 / R);
  };
  const size_t small = (size_t)255 << 20;
  int flip = 0;
  auto run = [&](const char* nm, auto kern) {
    timeit([&] {
      const uint8_t* b0 = buf + (flip ? small : 0);
      flip ^= 1;
      kern(b0);
    }, nm, (double)small);
  };
  for (int work : {0, 4, 8}) {
    char nm[128];
    snprintf(nm, sizeof nm, "ring PD=3 interleaved work=%d", work);
    run(nm, [&](const uint8_t* b0) { ring_stream<3><<<sms, 512>>>(b0, small, work, out); });
    snprintf(nm, sizeof nm, "batch U=2 DB interleaved work=%d", work);
    run(nm, [&](const uint8_t* b0) { batch_stream<2, true, false><<<sms, 512>>>(b0, small, work, out); });
    snprintf(nm, sizeof nm, "batch U=2 DB contiguous work=%d", work);
    run(nm, [&](const uint8_t* b0) { batch_stream<2, true, true><<<sms, 512>>>(b0, small, work, out); });
    snprintf(nm, sizeof nm, "batch U=3 noDB interleaved work=%d", work);
    run(nm, [&](const uint8_t* b0) { batch_stream<3, false, false><<<sms, 512>>>(b0, small, work, out); });
    snprintf(nm, sizeof nm, "batch U=3 noDB contiguous work=%d", work);
    run(nm, [&](const uint8_t* b0) { batch_stream<3, false, true><<<sms, 512>>>(b0, small, work, out); });
    snprintf(nm, sizeof nm, "batch U=4 noDB contiguous work=%d", work);
    run(nm, [&](const uint8_t* b0) { batch_stream<4, false, true><<<sms, 512>>>(b0, small, work, out); });
  }
  // a 255 MB stream (the fc1 q=3 g=128 weight), alternating two buffers so L2 never holds it
  for (int U : {4, 8}) {
    const size_t small = (size_t)255 << 20;
    char nm[128];
    snprintf(nm, sizeof nm, "255MB x2 alternating ldg.128 U=%d grid=%d", U, sms);
    int flip = 0;
    timeit([&] {
      const uint8_t* b0 = buf + (flip ? small : 0);
      flip ^= 1;
      if (U == 4) stream_ldg<4><<<sms, 512>>>(b0, small, 0, out);
      else stream_ldg<8><<<sms, 512>>>(b0, small, 0, out);
    }, nm, (double)small);
  }
  for (int ctas_per_sm : {1, 2}) {
    for (int pf : {0, 65536, 262144}) {
      char nm[128];
      snprintf(nm, sizeof nm, "ldg.128 U=4 grid=%dx%d pf=%dKB", sms, ctas_per_sm, pf / 1024);
      timeit([&] { stream_ldg<4><<<sms * ctas_per_sm, 512>>>(buf, bytes, pf, out); }, nm, (double)bytes);
      snprintf(nm, sizeof nm, "ldg.128 U=8 grid=%dx%d pf=%dKB", sms, ctas_per_sm, pf / 1024);
      timeit([&] { stream_ldg<8><<<sms * ctas_per_sm, 512>>>(buf, bytes, pf, out); }, nm, (double)bytes);
    }
  }
  CK(cudaFuncSetAttribute(lds_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072));
  const int iters = 4096;
  cudaEventRecord(a);
  lds_rate<<<sms, 512, 131072>>>(iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double lookups = (double)sms * 512 * iters * 16;
  printf("conflict-free LDS lookups: %.3e /s  (%.2f warp-LDS per SM-cycle at 1.965 GHz)\n", lookups / (ms * 1e-3),
         lookups / 32 / sms / (ms * 1e-3) / 1.965e9);
  CK(cudaGetLastError());
  return 0;
}
