// lutgemm_gemv_ep.cu -- the LUT-GEMV instantiations with the fused tensor-parallel epilogue (lutgemm_p2p.cu): MODE 1 of
// gemv_kernel.cuh, in their own translation unit so they compile in parallel with the others.
#include "gemv_kernel.cuh"

namespace lg {

cudaError_t launch_gemv_ep(const KParams& p, int grid, cudaStream_t st) {
  return dispatch_qz<GemvLaunchMode<1>::template F>(p, grid, st);
}

}  // namespace lg
