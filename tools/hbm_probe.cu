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
