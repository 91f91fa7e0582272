// quantize_kernels.cu -- offline quantizers producing the sources of
// lutgemm_pack_bcq from a dense fp16 weight (the step before
// the LUT-GEMM path).
//
//  * RTN: uniform min-max round-to-nearest per (row, group) -- the RTN baseline
//    of the paper's Tables 3/6; its (codes, s, z_hat) feed the App. C
//    conversion of the UNIFORM pack source.
//  * BCQ: w ~ sum_i alpha_i b_i (Sec. 2.3), greedy residual fit
//    (b_i = sign(r), alpha_i = mean|r|), then `iters` rounds of the alternating
//    solver App. E names (Xu et al.): alpha by least squares for fixed
//    signs, then every element's sign pattern = the nearest of the 2^q levels.
//
// One warp per (row, group); lane l owns the group's elements l, l+32, ...  The
// integer decisions (codes, signs, nearest level) are taken in the precision
// and operation order DESIGN.md states for them (fixed lane/butterfly fp32
// sums, fp16-stored scales used in the residual, fp64 elimination without
// fused multiply-adds), so the results are reproducible bit for bit.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "layout.cuh"
#include "lutgemm_internal.h"

namespace lg {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float wval(const __half* W, size_t idx) { return __half2float(W[idx]); }

// fixed-order fp32 sum over the warp: per-lane partial (sequential), then the
// butterfly p += shfl_xor(p, o), o = 16..1 (every lane ends with the same value)
__device__ __forceinline__ float butterfly_sum(float p) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) p += __shfl_xor_sync(kFull, p, o);
  return p;
}

__global__ void __launch_bounds__(256) quantize_rtn_kernel(const __half* __restrict__ W, int m, int n, int q, int g,
                                                           uint8_t* __restrict__ codes, __half* __restrict__ scale,
                                                           __half* __restrict__ zero) {
  const int G = n / g;
  const long long wid = (long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (wid >= (long long)m * G) return;
  const int lane = threadIdx.x & 31;
  const int row = (int)(wid / G), grp = (int)(wid % G);
  const size_t base = (size_t)row * n + (size_t)grp * g;
  float mn = 3.0e38f, mx = -3.0e38f;
  for (int t = lane; t < g; t += 32) {
    const float w = wval(W, base + t);
    mn = fminf(mn, w);
    mx = fmaxf(mx, w);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
  }
  const float top = (float)((1 << q) - 1);
  const __half z16 = __float2half_rn(mn);
  const bool flat = mx == mn;  // constant group: s = 1, codes 0, z_hat = min
  const __half s16 = flat ? __float2half_rn(1.f) : __float2half_rn(__fdiv_rn(__fsub_rn(mx, mn), top));
  const float z = __half2float(z16), s = __half2float(s16);
  for (int t = lane; t < g; t += 32) {
    float c = 0.f;
    if (!flat) c = fminf(fmaxf(rintf(__fdiv_rn(__fsub_rn(wval(W, base + t), z), s)), 0.f), top);
    codes[base + t] = (uint8_t)c;
  }
  if (lane == 0) {
    scale[(size_t)row * G + grp] = s16;
    zero[(size_t)row * G + grp] = z16;
  }
}

// sign word k of plane i of the warp's group (smem: [q][K] words, bit j <-> element 32k + j)
struct SignWords {
  uint32_t* w;
  int K;
  __device__ __forceinline__ bool bit(int i, int t) const { return (w[i * K + (t >> 5)] >> (t & 31)) & 1u; }
};

// residual of element t after planes < upto: r = w -/+ alpha_j, j = 0.. in order (fp32)
__device__ __forceinline__ float residual(float w, const SignWords& sw, const float* a, int upto, int t) {
  float r = w;
  for (int j = 0; j < upto; ++j) r = sw.bit(j, t) ? __fsub_rn(r, a[j]) : __fadd_rn(r, a[j]);
  return r;
}

__global__ void quantize_bcq_kernel(const __half* __restrict__ W, int m, int n, int q, int g, int iters,
                                    uint32_t* __restrict__ planes, __half* __restrict__ alpha_out) {
  extern __shared__ uint32_t qsm[];
  const int G = n / g, K = g / 32, L = 1 << q;
  const int wpb = blockDim.x / 32, wib = threadIdx.x / 32;
  const long long wid = (long long)blockIdx.x * wpb + wib;
  const int lane = threadIdx.x & 31;
  // per warp: q*K sign words, then 2^q fp32 levels
  uint32_t* mine = qsm + (size_t)wib * (q * K + L);
  SignWords sw{mine, K};
  float* lev = reinterpret_cast<float*>(mine + q * K);
  if (wid >= (long long)m * G) return;
  const int row = (int)(wid / G), grp = (int)(wid % G);
  const size_t base = (size_t)row * n + (size_t)grp * g;
  float a[8];
  __half a16[8];

  // ---- greedy: b_i = sign(r) (sign(0) = +1), alpha_i = fp16(mean |r|), r -= alpha_i b_i
  for (int i = 0; i < q; ++i) {
    float p = 0.f;
    for (int t = lane; t < g; t += 32) p = __fadd_rn(p, fabsf(residual(wval(W, base + t), sw, a, i, t)));
    const float S = butterfly_sum(p);
    a16[i] = __float2half_rn(__fdiv_rn(S, (float)g));
    a[i] = __half2float(a16[i]);
    for (int k = 0; k < K; ++k) {
      const int t = 32 * k + lane;
      const bool b = residual(wval(W, base + t), sw, a, i, t) >= 0.f;
      const uint32_t word = __ballot_sync(kFull, b);
      if (lane == 0) mine[i * K + k] = word;
    }
    __syncwarp();
  }

  // ---- alternating rounds
  for (int it = 0; it < iters; ++it) {
    // (a) alpha = argmin ||w - B alpha||: G = B^T B (integers), c = B^T w (fixed-order fp32 sums),
    //     Gaussian elimination in fp64 without pivoting, no fused multiply-adds
    double A[8][8], c[8];
    for (int i = 0; i < q; ++i) {
      for (int j = 0; j < q; ++j) {
        int agree = 0;
        for (int k = lane; k < K; k += 32) agree += __popc(~(mine[i * K + k] ^ mine[j * K + k]));
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) agree += __shfl_xor_sync(kFull, agree, o);
        A[i][j] = (double)(2 * agree - g);
      }
      float p = 0.f;
      for (int t = lane; t < g; t += 32) {
        const float w = wval(W, base + t);
        p = __fadd_rn(p, sw.bit(i, t) ? w : -w);
      }
      c[i] = (double)butterfly_sum(p);
    }
    bool singular = false;
    for (int kk = 0; kk < q && !singular; ++kk) {
      const double piv = A[kk][kk];
      if (!(piv > 0.5)) {
        singular = true;
        break;
      }
      for (int i = kk + 1; i < q; ++i) {
        const double f = __ddiv_rn(A[i][kk], piv);
        for (int j = kk; j < q; ++j) A[i][j] = __dsub_rn(A[i][j], __dmul_rn(f, A[kk][j]));
        c[i] = __dsub_rn(c[i], __dmul_rn(f, c[kk]));
      }
    }
    if (!singular) {
      double x[8];
      for (int i = q - 1; i >= 0; --i) {
        double acc = c[i];
        for (int j = i + 1; j < q; ++j) acc = __dsub_rn(acc, __dmul_rn(A[i][j], x[j]));
        x[i] = __ddiv_rn(acc, A[i][i]);
      }
      for (int i = 0; i < q; ++i) {
        a16[i] = __double2half(x[i]);
        a[i] = __half2float(a16[i]);
      }
    }
    // (b) levels v_k = sum_i (bit_i(k) ? +a_i : -a_i) in plane order (fp32); nearest level per element,
    //     lowest k on ties
    for (int k = lane; k < L; k += 32) {
      float v = 0.f;
      for (int i = 0; i < q; ++i) v = ((k >> i) & 1) ? __fadd_rn(v, a[i]) : __fsub_rn(v, a[i]);
      lev[k] = v;
    }
    __syncwarp();
    for (int kw = 0; kw < K; ++kw) {
      const int t = 32 * kw + lane;
      const float w = wval(W, base + t);
      int best = 0;
      float be = fabsf(__fsub_rn(w, lev[0]));
      for (int k = 1; k < L; ++k) {
        const float e = fabsf(__fsub_rn(w, lev[k]));
        if (e < be) {
          be = e;
          best = k;
        }
      }
      for (int i = 0; i < q; ++i) {
        const uint32_t word = __ballot_sync(kFull, (best >> i) & 1);
        if (lane == 0) mine[i * K + kw] = word;
      }
    }
    __syncwarp();
  }

  // ---- outputs: canonical planes [q][m][n/32] and alpha [m][G][q]
  for (int i = 0; i < q; ++i)
    for (int k = lane; k < K; k += 32) planes[((size_t)i * m + row) * (n / 32) + (size_t)grp * K + k] = mine[i * K + k];
  if (lane < q) alpha_out[((size_t)row * G + grp) * q + lane] = a16[lane];
}

inline unsigned blocks_of(long long warps, int wpb) { return (unsigned)((warps + wpb - 1) / wpb); }

}  // namespace

cudaError_t run_quantize_rtn(const uint16_t* W, int m, int n, int q, int g, uint8_t* codes, uint16_t* scale,
                             uint16_t* zero, cudaStream_t st) {
  const long long warps = (long long)m * (n / g);
  quantize_rtn_kernel<<<blocks_of(warps, 8), 256, 0, st>>>(reinterpret_cast<const __half*>(W), m, n, q, g, codes,
                                                          reinterpret_cast<__half*>(scale),
                                                          reinterpret_cast<__half*>(zero));
  return cudaGetLastError();
}

size_t quantize_bcq_smem_per_warp(int q, int g) { return ((size_t)q * (g / 32) + ((size_t)1 << q)) * 4u; }

cudaError_t run_quantize_bcq(const uint16_t* W, int m, int n, int q, int g, int iters, uint32_t* planes,
                             uint16_t* alpha, cudaStream_t st) {
  const size_t per = quantize_bcq_smem_per_warp(q, g);
  int wpb = (int)(49152 / per);
  wpb = wpb < 1 ? 1 : (wpb > 8 ? 8 : wpb);
  const size_t smem = per * wpb;
  cudaError_t e = cudaFuncSetAttribute(quantize_bcq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long warps = (long long)m * (n / g);
  quantize_bcq_kernel<<<blocks_of(warps, wpb), 32 * wpb, smem, st>>>(reinterpret_cast<const __half*>(W), m, n, q, g,
                                                                    iters, planes, reinterpret_cast<__half*>(alpha));
  return cudaGetLastError();
}

}  // namespace lg
