// pack_kernels.cu -- offline repacking into the kernel-native layout (layout.cuh).
//
// BCQ source: canonical planes/alpha/offset are permuted into the record
// stream of layout.cuh, bit for bit.
// UNIFORM source: App. C -- plane i bit = bit i of the code
// (b_i = 2 b_hat_i - 1), alpha_i = 2^(i-1) s (exact power-of-two
// scaling of an fp16 s), z = sum_i alpha_i + z_hat summed in fp64 and rounded
// once to fp16 (R17).  The compact format stores s instead of the q alphas.  Offline and untimed ("two-step methodology").
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

__global__ void pack_keys_kernel(const uint32_t* __restrict__ src, uint8_t* __restrict__ dst, Shape sh) {
  const int nw = (sh.n + 31) / 32;
  const size_t total = (size_t)sh.q * sh.m4 * nw;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int w = (int)(idx % nw);
    const int r = (int)((idx / nw) % sh.m4);
    const int i = (int)(idx / ((size_t)nw * sh.m4));
    const uint32_t v = r < sh.m ? src[((size_t)i * sh.m + r) * nw + w] : 0u;
    const int s = w / kLanesPerSlice, p = w % kLanesPerSlice;
    const int Ls = slice_lanes(sh.n, s);
    *reinterpret_cast<uint32_t*>(dst + key_at(sh, s, Ls, r / 4, i, p, r % 4)) = v;
  }
}

__global__ void unpack_keys_kernel(const uint8_t* __restrict__ src, uint32_t* __restrict__ dst, Shape sh) {
  const int nw = (sh.n + 31) / 32;
  const size_t total = (size_t)sh.q * sh.m * nw;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int w = (int)(idx % nw);
    const int r = (int)((idx / nw) % sh.m);
    const int i = (int)(idx / ((size_t)nw * sh.m));
    const int s = w / kLanesPerSlice, p = w % kLanesPerSlice;
    const int Ls = slice_lanes(sh.n, s);
    dst[idx] = *reinterpret_cast<const uint32_t*>(src + key_at(sh, s, Ls, r / 4, i, p, r % 4));
  }
}

// scales: one thread per (slice, row quad, slice-local group k); writes alpha
// for all q planes and z (canonical alpha [m][G][q], z [m][G]).
__global__ void pack_scales_kernel(const uint16_t* __restrict__ alpha, const uint16_t* __restrict__ offset,
                                   uint8_t* __restrict__ dst, Shape sh) {
  const int gmax = slice_groups(sh, kLanesPerSlice);
  const size_t total = (size_t)sh.S * sh.RQ * gmax;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx % gmax);
    const int rq = (int)((idx / gmax) % sh.RQ);
    const int s = (int)(idx / ((size_t)gmax * sh.RQ));
    const int Ls = slice_lanes(sh.n, s);
    if (k >= slice_groups(sh, Ls)) continue;
    const int grp = global_group(sh, s, k);
    if (grp >= sh.G) continue;  // unused entry (kGrpSpan bound, kGrpChunk chunks past n): stays zero
    for (int r4 = 0; r4 < 4; ++r4) {
      const int r = 4 * rq + r4;
      for (int i = 0; i < sh.q; ++i)
        *reinterpret_cast<uint16_t*>(dst + alpha_at(sh, s, Ls, rq, i, k, r4)) =
            r < sh.m ? alpha[((size_t)r * sh.G + grp) * sh.q + i] : (uint16_t)0;
      if (sh.has_z)
        *reinterpret_cast<uint16_t*>(dst + z_at(sh, s, Ls, rq, k, r4)) =
            (r < sh.m && offset) ? offset[(size_t)r * sh.G + grp] : (uint16_t)0;
    }
  }
}

__global__ void unpack_scales_kernel(const uint8_t* __restrict__ src, uint16_t* __restrict__ alpha,
                                     uint16_t* __restrict__ offset, Shape sh) {
  const size_t total = (size_t)sh.m * sh.G;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int grp = (int)(idx % sh.G);
    const int r = (int)(idx / sh.G);
    int s, k;
    home_of_group(sh, grp, &s, &k);
    const int Ls = slice_lanes(sh.n, s);
    if (alpha && sh.compact) {  // alpha_i = 2^(i-1) s
      const double sv = (double)__half2float(
          __ushort_as_half(*reinterpret_cast<const uint16_t*>(src + alpha_at(sh, s, Ls, r / 4, 0, k, r % 4))));
      for (int i = 0; i < sh.q; ++i) alpha[idx * sh.q + i] = __half_as_ushort(__double2half(ldexp(sv, i - 1)));
    } else if (alpha) {
      for (int i = 0; i < sh.q; ++i)
        alpha[idx * sh.q + i] = *reinterpret_cast<const uint16_t*>(src + alpha_at(sh, s, Ls, r / 4, i, k, r % 4));
    }
    if (offset && sh.has_z)
      offset[idx] = *reinterpret_cast<const uint16_t*>(src + z_at(sh, s, Ls, r / 4, k, r % 4));
  }
}

// uniform codes [m][n] -> keys: plane i word = bit i of 32 codes (b_hat_i, App. C)
__global__ void pack_uniform_keys_kernel(const uint8_t* __restrict__ codes, uint8_t* __restrict__ dst, Shape sh) {
  const int nw = (sh.n + 31) / 32;
  const size_t total = (size_t)sh.m4 * nw;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int w = (int)(idx % nw);
    const int r = (int)(idx / nw);
    uint32_t words[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (r < sh.m) {
      const uint8_t* c = codes + (size_t)r * sh.n + 32 * w;
      const int nc = min(32, sh.n - 32 * w);  // the last word may be partial (n % 32 != 0): padding bits 0
      for (int j = 0; j < nc; ++j) {
        const uint32_t code = c[j];
        for (int i = 0; i < sh.q; ++i) words[i] |= ((code >> i) & 1u) << j;
      }
    }
    const int s = w / kLanesPerSlice, p = w % kLanesPerSlice;
    const int Ls = slice_lanes(sh.n, s);
    for (int i = 0; i < sh.q; ++i) *reinterpret_cast<uint32_t*>(dst + key_at(sh, s, Ls, r / 4, i, p, r % 4)) = words[i];
  }
}

// alpha_i = 2^(i-1) s ; z = sum_i alpha_i + z_hat  (App. C Eq. 8), per (slice, rq, k)
__global__ void pack_uniform_scales_kernel(const uint16_t* __restrict__ scale, const uint16_t* __restrict__ zero,
                                           uint8_t* __restrict__ dst, Shape sh) {
  const int gmax = slice_groups(sh, kLanesPerSlice);
  const size_t total = (size_t)sh.S * sh.RQ * gmax;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx % gmax);
    const int rq = (int)((idx / gmax) % sh.RQ);
    const int s = (int)(idx / ((size_t)gmax * sh.RQ));
    const int Ls = slice_lanes(sh.n, s);
    if (k >= slice_groups(sh, Ls)) continue;
    const int grp = global_group(sh, s, k);
    if (grp >= sh.G) continue;  // unused entry: stays zero
    for (int r4 = 0; r4 < 4; ++r4) {
      const int r = 4 * rq + r4;
      double sv = 0.0, zh = 0.0;
      if (r < sh.m) {
        sv = (double)__half2float(__ushort_as_half(scale[(size_t)r * sh.G + grp]));
        zh = (double)__half2float(__ushort_as_half(zero[(size_t)r * sh.G + grp]));
      }
      double sum_alpha = 0.0;
      for (int i = 0; i < sh.q; ++i) {
        const double a = ldexp(sv, i - 1);
        sum_alpha += a;
        if (!sh.compact)
          *reinterpret_cast<uint16_t*>(dst + alpha_at(sh, s, Ls, rq, i, k, r4)) = __half_as_ushort(__double2half(a));
      }
      if (sh.compact)  // the compact format stores s itself (alpha_i = 2^(i-1) s derived in-kernel)
        *reinterpret_cast<uint16_t*>(dst + alpha_at(sh, s, Ls, rq, 0, k, r4)) =
            r < sh.m ? scale[(size_t)r * sh.G + grp] : (uint16_t)0;
      *reinterpret_cast<uint16_t*>(dst + z_at(sh, s, Ls, rq, k, r4)) =
          __half_as_ushort(__double2half(r < sh.m ? sum_alpha + zh : 0.0));
    }
  }
}

}  // namespace

cudaError_t run_pack_bcq(const Shape& sh, const uint32_t* planes, const uint16_t* alpha, const uint16_t* offset,
                         void* dst, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(dst, 0, packed_bytes(sh), st);
  if (e != cudaSuccess) return e;
  pack_keys_kernel<<<blocks_for((size_t)sh.q * sh.m4 * ((sh.n + 31) / 32)), kPackThreads, 0, st>>>(
      planes, static_cast<uint8_t*>(dst), sh);
  pack_scales_kernel<<<blocks_for((size_t)sh.S * sh.RQ * slice_groups(sh, kLanesPerSlice)), kPackThreads, 0, st>>>(
      alpha, offset, static_cast<uint8_t*>(dst), sh);
  return cudaGetLastError();
}

cudaError_t run_pack_uniform(const Shape& sh, const uint8_t* codes, const uint16_t* scale, const uint16_t* zero,
                             void* dst, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(dst, 0, packed_bytes(sh), st);
  if (e != cudaSuccess) return e;
  pack_uniform_keys_kernel<<<blocks_for((size_t)sh.m4 * ((sh.n + 31) / 32)), kPackThreads, 0, st>>>(
      codes, static_cast<uint8_t*>(dst), sh);
  pack_uniform_scales_kernel<<<blocks_for((size_t)sh.S * sh.RQ * slice_groups(sh, kLanesPerSlice)), kPackThreads, 0,
                               st>>>(scale, zero, static_cast<uint8_t*>(dst), sh);
  return cudaGetLastError();
}

cudaError_t run_unpack(const Shape& sh, const void* src, uint32_t* planes, uint16_t* alpha, uint16_t* offset,
                       cudaStream_t st) {
  if (planes)
    unpack_keys_kernel<<<blocks_for((size_t)sh.q * sh.m * ((sh.n + 31) / 32)), kPackThreads, 0, st>>>(
        static_cast<const uint8_t*>(src), planes, sh);
  if (alpha || offset)
    unpack_scales_kernel<<<blocks_for((size_t)sh.m * sh.G), kPackThreads, 0, st>>>(static_cast<const uint8_t*>(src),
                                                                                  alpha, offset, sh);
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
