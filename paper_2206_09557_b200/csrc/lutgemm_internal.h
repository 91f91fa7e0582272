// lutgemm_internal.h -- declarations shared by the kernel and ABI translation units.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "layout.cuh"

namespace lg {

constexpr int kFusedMaxJ = 256;  // max CTAs per slice in the fused-reduction mode

// the layout constants of a full (32-lane) slice, computed once on the host so the kernels' prologue
// does not re-derive them (layout.cuh)
struct FullSlice {
  unsigned long long stride;  // bytes per slice
  unsigned long long aoff;    // offset of the alpha region in a slice
  unsigned long long zoff;    // offset of the z region
  uint32_t KB, AB, ZB;        // bytes per row quad of each region
};

__host__ __device__ inline FullSlice full_slice(const Shape& sh) {
  FullSlice f;
  f.KB = keys_bytes(sh, kLanesPerSlice);
  f.AB = alpha_bytes(sh, kLanesPerSlice);
  f.ZB = z_bytes(sh, kLanesPerSlice);
  f.stride = slice_bytes(sh, kLanesPerSlice);
  f.aoff = pad256((size_t)sh.RQ * f.KB);
  f.zoff = f.aoff + pad256((size_t)sh.RQ * f.AB);
  return f;
}

struct KParams {
  const uint8_t* data;   // packed record stream (layout.cuh)
  const __half* x;   // [b][n]
  __half* y;         // [b][m] fp16 output (or null)
  float* yf;         // [b][m] fp32 output (or null)
  float* partial;    // [S][b][m4] split-K partials
  unsigned* counters;  // GEMV fused mode: arrive/depart counters per row-quad group (zero between launches)
  Shape sh;
  FullSlice fs;      // full_slice(sh)
  int b;
  int bl;            // batched: log2 of the padded batch b_pad >= b (partials are [S2][m4][b_pad])
  int nv;            // batched: V-wide batch vectors per table entry slot group (b_pad = V * nv)
  int spi;           // batched: LUT slices per work item (split-K factor S2 = ceil(S / spi))
  int qpw;           // batched: row quads per work item (256 or 128)
  int fused_J;       // GEMV: CTAs per slice in the fused-reduction mode (0: separate reduction kernel);
                     // CTA c runs slice c / J, row group c % J
  float rcp_J;       // fused mode: 1 / J (fused_slot: the division without an integer divide)
  int gq[kFusedMaxJ + 1];  // fused mode: first unit (row quad / quad group) of row group fj, gq[J] = units
                     // (host-computed: no division in the kernels' prologue)
  int smem_bytes;    // dynamic shared memory per CTA (0: kSmemBytesBase)
  int xdirect;       // GEMV: each thread loads its 8 x values for the LUT build straight from global memory
                     // (0: the slice is staged into shared memory by the bulk-copy engine first)
  int reducers;      // GEMV fused mode: the last R CTAs to arrive in a row-quad group reduce it
  // fused tensor-parallel epilogue over peer memory (NEXT-1, lutgemm_p2p.cu, gemv_kernel.cuh
  // p2p_epilogue): LL words (data | stamp << 32) into the ranks' windows.  p2p_mode 1 (rows
  // all-gather): rows (r, r+1) of the gathered output at window[par][pr] + 4 (yoff + r);
  // p2p_mode 2 (column split): the fp32 row r at its owner o = r / p2p_mb, slot [self][r - o mb]
  // (8-byte words), the owner's fp16 rows (r, r+1) at p2p_yarea + 4 r.  par = *p2p_round & 1
  // (device-side round: graph-capturable), stamp = low 32 bits of *p2p_round + 1.
  uint8_t* p2p_win[2][8];
  const unsigned long long* p2p_round;
  int p2p_mode;      // 0: plain output
  unsigned long long p2p_timeout_ns;  // an LL wait longer than this traps (LUTGEMM_P2P_TIMEOUT_MS, default 30 s)
  int npeers;
  int yoff;
  int p2p_self;
  int p2p_mb;
  unsigned p2p_yarea;
  int s2;            // b <= 4 GEMV-structured kernel: number of sub-slices (0: not used)
  long long items;
  unsigned long long* trace;  // optional per-CTA timeline (kTraceSlots u64 per CTA), or null
};

constexpr int kTraceSlots = 8;
// tracing (debug): enable a per-CTA %globaltimer timeline of the next launches
void trace_enable(int on);
size_t trace_read(unsigned long long* host, size_t n);

size_t workspace_bytes(const Shape& sh, int b);
// product kernels (LUT + reduction) this process has launched
unsigned long long launch_count();
// padded batch of the batched kernel's partials (1 for the GEMV)
int batch_pad(int b);

// y (fp16) or yf (fp32) [b][m] = X [b][n] W^T.  Two launches chained with
// programmatic dependent launch: the LUT kernel (split-K partials), then the
// fixed-order cross-slice reduction.
cudaError_t run_product(const Shape& sh, const void* data, const uint16_t* x, int b, uint16_t* y, float* yf,
                        void* ws, cudaStream_t st);

// NEXT-1: b = 1 product whose fused reduction stores the rows into the ranks' windows (see
// KParams::p2p_*), exchanges with every rank and writes the full result to y; requires the fused
// GEMV mode (returns cudaErrorNotSupported otherwise).
struct P2PArgs {
  uint8_t* win[2][8];
  const unsigned long long* round;
  int mode, npeers, self, yoff, mb;
  unsigned yarea;
};
cudaError_t run_gemv_p2p(const Shape& sh, const void* data, const uint16_t* x, void* ws, const P2PArgs& a,
                         uint16_t* y, cudaStream_t st);

cudaError_t run_pack_bcq(const Shape& sh, const uint32_t* planes, const uint16_t* alpha, const uint16_t* offset,
                         void* dst, cudaStream_t st);
cudaError_t run_pack_uniform(const Shape& sh, const uint8_t* codes, const uint16_t* scale, const uint16_t* zero,
                             void* dst, cudaStream_t st);
cudaError_t run_unpack(const Shape& sh, const void* src, uint32_t* planes, uint16_t* alpha, uint16_t* offset,
                       cudaStream_t st);

// quantizers: dense fp16 W [m][n] -> canonical pack sources
cudaError_t run_quantize_rtn(const uint16_t* W, int m, int n, int q, int g, uint8_t* codes, uint16_t* scale,
                             uint16_t* zero, cudaStream_t st);
cudaError_t run_quantize_bcq(const uint16_t* W, int m, int n, int q, int g, int iters, uint32_t* planes,
                             uint16_t* alpha, cudaStream_t st);
size_t quantize_bcq_smem_per_warp(int q, int g);

// TP helpers
cudaError_t run_cast_f32_f16(const float* src, uint16_t* dst, size_t count, cudaStream_t st);
// src [P][b][ms] -> dst [b][P*ms]
cudaError_t run_gather_permute(const uint16_t* src, uint16_t* dst, int P, int b, int ms, cudaStream_t st);

}  // namespace lg
