// lutgemm_gemv.cu -- the plain LUT-GEMV instantiations (MODE 0, gemv_kernel.cuh), the mode
// dispatch, and the cross-slice reduction kernel of the non-fused mode.
#include "gemv_kernel.cuh"

namespace lg {

// ---------------------------------------------------------------------------
// Cross-slice reduction: Y[beta][r] = sum_{s=0}^{S-1} partial[s][beta][r] in
// slice order (deterministic, R11), then fp16 round-to-nearest-even (or fp32).
// One thread per (beta, row pair), up to 32 slices per L2 round trip (the split
// path of wide layers has S up to ~200 sub-slices); launched with PDL after the
// LUT kernel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lut_reduce_kernel(const float* __restrict__ partial, int S, int b, int m,
                                                         int m4, __half* __restrict__ y, float* __restrict__ yf) {
  pdl_launch_dependents();  // the next product may start streaming its weights
  pdl_wait();               // partials are complete and visible
  const int RP = m4 / 2;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= b * RP) return;
  const int beta = idx / RP, rp = idx % RP;
  const float2* src = reinterpret_cast<const float2*>(partial + (size_t)beta * m4) + rp;
  const size_t stride = (size_t)b * RP;  // float2 units between slices
  float2 acc = make_float2(0.f, 0.f);
  for (int s0 = 0; s0 < S; s0 += 32) {
    float2 v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = (s0 + k < S) ? __ldcg(src + (size_t)(s0 + k) * stride) : make_float2(0, 0);
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (s0 + k < S) {
        acc.x += v[k].x;
        acc.y += v[k].y;
      }
  }
  const float r[2] = {acc.x, acc.y};
  const int row0 = 2 * rp;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (row0 + k < m) {
      const size_t o = (size_t)beta * m + row0 + k;
      if (yf) yf[o] = r[k];
      else y[o] = __float2half_rn(r[k]);
    }
  }
}


cudaError_t launch_gemv(const KParams& p, int grid, cudaStream_t st) {
  if (p.p2p_mode != 0) return launch_gemv_ep(p, grid, st);
  return dispatch_qz<GemvLaunchMode<0>::template F>(p, grid, st);
}

cudaError_t launch_reduce(const KParams& p, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static bool attr_set = false;
  if (!attr_set) {  // keep the max-shared-memory carveout: no L1/smem reconfiguration between the two kernels
    cudaFuncSetAttribute(lut_reduce_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr_set = true;
  }
  const int threads = 256;
  const int total = p.b * (p.sh.m4 / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((total + threads - 1) / threads);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cfg.attrs = const_cast<cudaLaunchAttribute*>(pdl_attr());
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lut_reduce_kernel, (const float*)p.partial, p.sh.S, p.b, p.sh.m, p.sh.m4, p.y,
                            p.yf);
}

}  // namespace lg
