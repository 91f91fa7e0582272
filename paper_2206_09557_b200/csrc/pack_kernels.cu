// pack_kernels.cu -- offline repacking into the kernel-native layout (layout.cuh).
//
// BCQ source: canonical planes/alpha/offset are permuted, bit for bit.
// UNIFORM source: App. C -- plane i bit = bit i of the code
// (b_i = 2 b_hat_i - 1), alpha_i = 2^(i-1) s (exact power-of-two
// scaling of an fp16 s), z = sum_i alpha_i + z_hat summed in fp64 and rounded
// once to fp16 (R17).  Offline and untimed ("two-step methodology").
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "layout.cuh"
#include "lutgemm_internal.h"

namespace lg {

namespace {

constexpr int kPackThreads = 256;

inline int blocks_for(size_t total) {
  size_t b = (total + kPackThreads - 1) / kPackThreads;
  return (int)(b > 65535u * 16u ? 65535u * 16u : (b ? b : 1));
}

__global__ void pack_planes_kernel(const uint32_t* __restrict__ src, uint8_t* __restrict__ dst, Shape sh) {
  const int nw = sh.n / 32;
  const size_t total = (size_t)sh.q * sh.m4 * nw;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int w = (int)(idx % nw);
    const int r = (int)((idx / nw) % sh.m4);
    const int i = (int)(idx / ((size_t)nw * sh.m4));
    const uint32_t v = r < sh.m ? src[((size_t)i * sh.m + r) * nw + w] : 0u;
    const int s = w / kLanesPerSlice, p = w % kLanesPerSlice;
    const int Ls = slice_lanes(sh.n, s);
    *reinterpret_cast<uint32_t*>(dst + plane_vec_offset(sh, s, Ls, r / 4, i, p) + (r % 4) * 4) = v;
  }
}

__global__ void unpack_planes_kernel(const uint8_t* __restrict__ src, uint32_t* __restrict__ dst, Shape sh) {
  const int nw = sh.n / 32;
  const size_t total = (size_t)sh.q * sh.m * nw;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int w = (int)(idx % nw);
    const int r = (int)((idx / nw) % sh.m);
    const int i = (int)(idx / ((size_t)nw * sh.m));
    const int s = w / kLanesPerSlice, p = w % kLanesPerSlice;
    const int Ls = slice_lanes(sh.n, s);
    dst[idx] = *reinterpret_cast<const uint32_t*>(src + plane_vec_offset(sh, s, Ls, r / 4, i, p) + (r % 4) * 4);
  }
}

// alpha canonical [m][G][q] <-> native [RQ][q][G][4]
__global__ void pack_alpha_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst, Shape sh) {
  const size_t total = alpha_elems(sh);
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int r4 = (int)(idx % 4);
    const int grp = (int)((idx / 4) % sh.G);
    const int i = (int)((idx / (4 * (size_t)sh.G)) % sh.q);
    const int rq = (int)(idx / (4 * (size_t)sh.G * sh.q));
    const int r = 4 * rq + r4;
    dst[idx] = r < sh.m ? src[((size_t)r * sh.G + grp) * sh.q + i] : (uint16_t)0;
  }
}

__global__ void unpack_alpha_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst, Shape sh) {
  const size_t total = (size_t)sh.m * sh.G * sh.q;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % sh.q);
    const int grp = (int)((idx / sh.q) % sh.G);
    const int r = (int)(idx / ((size_t)sh.q * sh.G));
    dst[idx] = src[alpha_index(sh, r / 4, i, grp, r % 4)];
  }
}

// offset canonical [m][G] <-> native [RQ][G][4]
__global__ void pack_offset_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst, Shape sh) {
  const size_t total = offset_elems(sh);
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int r4 = (int)(idx % 4);
    const int grp = (int)((idx / 4) % sh.G);
    const int rq = (int)(idx / (4 * (size_t)sh.G));
    const int r = 4 * rq + r4;
    dst[idx] = r < sh.m ? src[(size_t)r * sh.G + grp] : (uint16_t)0;
  }
}

__global__ void unpack_offset_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst, Shape sh) {
  const size_t total = (size_t)sh.m * sh.G;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int grp = (int)(idx % sh.G);
    const int r = (int)(idx / sh.G);
    dst[idx] = src[offset_index(sh, r / 4, grp, r % 4)];
  }
}

// uniform codes [m][n] -> native planes: plane i word = bit i of 32 codes
__global__ void pack_uniform_planes_kernel(const uint8_t* __restrict__ codes, uint8_t* __restrict__ dst, Shape sh) {
  const int nw = sh.n / 32;
  const size_t total = (size_t)sh.m4 * nw;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int w = (int)(idx % nw);
    const int r = (int)(idx / nw);
    uint32_t words[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (r < sh.m) {
      const uint8_t* c = codes + (size_t)r * sh.n + 32 * w;
      for (int j = 0; j < 32; ++j) {
        const uint32_t code = c[j];
        for (int i = 0; i < sh.q; ++i) words[i] |= ((code >> i) & 1u) << j;
      }
    }
    const int s = w / kLanesPerSlice, p = w % kLanesPerSlice;
    const int Ls = slice_lanes(sh.n, s);
    for (int i = 0; i < sh.q; ++i)
      *reinterpret_cast<uint32_t*>(dst + plane_vec_offset(sh, s, Ls, r / 4, i, p) + (r % 4) * 4) = words[i];
  }
}

// alpha_i = 2^(i-1) s ; z = sum_i alpha_i + z_hat  (App. C Eq. 8)
__global__ void pack_uniform_scales_kernel(const uint16_t* __restrict__ scale, const uint16_t* __restrict__ zero,
                                           uint16_t* __restrict__ alpha, uint16_t* __restrict__ offset, Shape sh) {
  const size_t total = offset_elems(sh);  // one thread per (rq, grp, r4)
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int r4 = (int)(idx % 4);
    const int grp = (int)((idx / 4) % sh.G);
    const int rq = (int)(idx / (4 * (size_t)sh.G));
    const int r = 4 * rq + r4;
    double s = 0.0, zh = 0.0;
    if (r < sh.m) {
      s = (double)__half2float(__ushort_as_half(scale[(size_t)r * sh.G + grp]));
      zh = (double)__half2float(__ushort_as_half(zero[(size_t)r * sh.G + grp]));
    }
    double sum_alpha = 0.0;
    for (int i = 0; i < sh.q; ++i) {
      const double a = ldexp(s, i - 1);
      sum_alpha += a;
      alpha[alpha_index(sh, rq, i, grp, r4)] = __half_as_ushort(__double2half(a));
    }
    offset[offset_index(sh, rq, grp, r4)] = __half_as_ushort(__double2half(r < sh.m ? sum_alpha + zh : 0.0));
  }
}

}  // namespace

cudaError_t run_pack_bcq(const Shape& sh, const uint32_t* planes, const uint16_t* alpha, const uint16_t* offset,
                         void* dplanes, void* dalpha, void* doffset, cudaStream_t st) {
  pack_planes_kernel<<<blocks_for((size_t)sh.q * sh.m4 * (sh.n / 32)), kPackThreads, 0, st>>>(
      planes, static_cast<uint8_t*>(dplanes), sh);
  pack_alpha_kernel<<<blocks_for(alpha_elems(sh)), kPackThreads, 0, st>>>(alpha, static_cast<uint16_t*>(dalpha), sh);
  if (offset && doffset)
    pack_offset_kernel<<<blocks_for(offset_elems(sh)), kPackThreads, 0, st>>>(offset, static_cast<uint16_t*>(doffset),
                                                                             sh);
  return cudaGetLastError();
}

cudaError_t run_pack_uniform(const Shape& sh, const uint8_t* codes, const uint16_t* scale, const uint16_t* zero,
                             void* dplanes, void* dalpha, void* doffset, cudaStream_t st) {
  pack_uniform_planes_kernel<<<blocks_for((size_t)sh.m4 * (sh.n / 32)), kPackThreads, 0, st>>>(
      codes, static_cast<uint8_t*>(dplanes), sh);
  pack_uniform_scales_kernel<<<blocks_for(offset_elems(sh)), kPackThreads, 0, st>>>(
      scale, zero, static_cast<uint16_t*>(dalpha), static_cast<uint16_t*>(doffset), sh);
  return cudaGetLastError();
}

cudaError_t run_unpack(const Shape& sh, const void* dplanes, const void* dalpha, const void* doffset,
                       uint32_t* planes, uint16_t* alpha, uint16_t* offset, cudaStream_t st) {
  if (planes)
    unpack_planes_kernel<<<blocks_for((size_t)sh.q * sh.m * (sh.n / 32)), kPackThreads, 0, st>>>(
        static_cast<const uint8_t*>(dplanes), planes, sh);
  if (alpha)
    unpack_alpha_kernel<<<blocks_for((size_t)sh.m * sh.G * sh.q), kPackThreads, 0, st>>>(
        static_cast<const uint16_t*>(dalpha), alpha, sh);
  if (offset && doffset)
    unpack_offset_kernel<<<blocks_for((size_t)sh.m * sh.G), kPackThreads, 0, st>>>(
        static_cast<const uint16_t*>(doffset), offset, sh);
  return cudaGetLastError();
}

namespace {
__global__ void cast_f32_f16_kernel(const float* __restrict__ src, __half* __restrict__ dst, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __float2half_rn(src[i]);
}
__global__ void gather_permute_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst, int P, int b,
                                      int ms) {
  const size_t total = (size_t)P * b * ms;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % ms);
    const int bt = (int)((i / ms) % b);
    const int rk = (int)(i / ((size_t)ms * b));
    dst[(size_t)bt * P * ms + (size_t)rk * ms + r] = src[i];
  }
}
}  // namespace

cudaError_t run_cast_f32_f16(const float* src, uint16_t* dst, size_t count, cudaStream_t st) {
  cast_f32_f16_kernel<<<blocks_for(count), kPackThreads, 0, st>>>(src, reinterpret_cast<__half*>(dst), count);
  return cudaGetLastError();
}

cudaError_t run_gather_permute(const uint16_t* src, uint16_t* dst, int P, int b, int ms, cudaStream_t st) {
  gather_permute_kernel<<<blocks_for((size_t)P * b * ms), kPackThreads, 0, st>>>(src, dst, P, b, ms);
  return cudaGetLastError();
}

}  // namespace lg
