// lutgemm_kernels.cu -- sm_100a LUT-GEMM kernels (GEMV b=1 and batched b<=32).
//
// Method: y = sum_i A_i o (B_i . x) (Sec. 3.2) plus the
// extended-BCQ bias (Eq. 3).  Every thread block (CTA) "first
// conducts pre-computation using partial x values ... to fill up the l number
// of LUTs" (App. B), threads then turn packed sign bits into table
// lookups, scales are applied once per (row, group, plane)
// (P:L586), and the CTAs' partial outputs are accumulated across the column
// slices -- here in a fixed order instead of atomicAdd (R11).
//
// B200 design:
//  * one persistent CTA per SM (512 threads, 16 warps), a balanced static
//    split of (slice, row-quad) work items;
//  * mu = 8, fp32 LUT entries, 128 tables x 256 entries = 128 KB of shared
//    memory per 1024-column slice, stored interleaved so that entry k of the
//    table used by lane l at chunk step j lives at
//        LUT + (j>>1)*64KB + k*256 + (32*(j&1) + l)*4
//    -> every lookup instruction of a warp hits 32 distinct banks whatever the
//    keys are (bank = lane), and key -> address is ONE byte permute (PRMT)
//    because the LUT sits on a 64 KB boundary of the shared window;
//  * packed planes streamed HBM -> registers with 128-bit coalesced loads
//    (L1::no_allocate), a PD-deep register ring prefetching row quads;
//  * the activation slice is staged into shared memory by the bulk-copy
//    (TMA) engine, double-buffered one segment ahead;
//  * per-row partials reduced in registers by a 6-shuffle transpose-reduce,
//    written to an fp32 split-K workspace, and summed in slice order by the
//    last CTA to finish each row block (deterministic, one launch).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "layout.cuh"
#include "lutgemm_internal.h"
#include "ptx.cuh"

namespace lg {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kBlkQuads = 64;      // GEMV arrival-counter block: 64 row quads = 256 rows
constexpr int kQPW = 8;            // batched: row quads per warp per work item
constexpr int kMiscBytes = 8192;   // x double buffer (2 x 2 KB) + mbarriers + flags
constexpr int kSmemBytes = 3 * 65536;  // LUT (128 KB) on a 64 KB boundary + misc, any base
constexpr unsigned kFull = 0xffffffffu;

struct SmemMap {
  uint32_t lut;     // shared-window address of the LUT (multiple of 64 KB)
  uint32_t misc;    // shared-window address of the misc block
  uint8_t* misc_p;  // generic pointer to the misc block
};

__device__ __forceinline__ SmemMap map_smem(uint8_t* smem) {
  SmemMap m;
  const uint32_t base = smem_u32(smem);
  m.lut = (base + 0xFFFFu) & ~0xFFFFu;
  m.misc = (m.lut - base >= (uint32_t)kMiscBytes) ? base : m.lut + kLutBytes;
  m.misc_p = smem + (m.misc - base);
  return m;
}

// Byte offset of table slot (lane l, chunk step j) inside the LUT.
__device__ __forceinline__ uint32_t table_offset(int l, int j) {
  return (uint32_t)(j >> 1) * 65536u + (uint32_t)(32 * (j & 1) + l) * 4u;
}

// Build entries [64h, 64h+64) of one table T[k] = sum_j (2 bit_j(k) - 1) x_j
// (mu = 8, key bit j <-> column 8t+j, R3).  T[k] = L[k&15] + H[k>>4]
// with L over x0..x3 and H over x4..x7: 1 add per entry (Eq. 2's C_build).
__device__ __forceinline__ void build_table_part(uint32_t tbl, const __half* xc, int h) {
  const uint4 raw = *reinterpret_cast<const uint4*>(xc);
  const float2 x01 = h2_to_f2(raw.x), x23 = h2_to_f2(raw.y), x45 = h2_to_f2(raw.z), x67 = h2_to_f2(raw.w);
  const float a[4] = {-x01.x - x01.y, x01.x - x01.y, -x01.x + x01.y, x01.x + x01.y};
  const float b[4] = {-x23.x - x23.y, x23.x - x23.y, -x23.x + x23.y, x23.x + x23.y};
  const float c[4] = {-x45.x - x45.y, x45.x - x45.y, -x45.x + x45.y, x45.x + x45.y};
  const float d = ((h & 1) ? x67.x : -x67.x) + ((h & 2) ? x67.y : -x67.y);
  float L[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) L[k] = a[k & 3] + b[k >> 2];
  const uint32_t base = tbl + (uint32_t)(64 * h) * 256u;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const float H = c[u] + d;
#pragma unroll
    for (int k = 0; k < 16; ++k) sts_f32(base + (uint32_t)(16 * u + k) * 256u, L[k] + H);
  }
}

// Four lookups (chunk steps j = 0..3 of one packed word = 4 keys) summed.
// lc = LUT[31:16] | (4l+128) << 8 | 4l ; PRMT puts key byte j in bits 8..15.
__device__ __forceinline__ float lut4(uint32_t w, uint32_t lc) {
  const float v0 = lds_f32<0>(prmt<0x7604>(w, lc));
  const float v1 = lds_f32<0>(prmt<0x7615>(w, lc));
  const float v2 = lds_f32<65536>(prmt<0x7624>(w, lc));
  const float v3 = lds_f32<65536>(prmt<0x7635>(w, lc));
  return (v0 + v1) + (v2 + v3);
}

// Transpose-reduce of 4 per-lane row partials over the 32 lanes; returns the
// full sum of row (lane >> 3) & 3 (valid in lanes 0, 8, 16, 24).
__device__ __forceinline__ float reduce4(const float acc[4], int lane) {
  const bool hi16 = lane & 16;
  const float s0 = hi16 ? acc[0] : acc[2], s1 = hi16 ? acc[1] : acc[3];
  float k0 = hi16 ? acc[2] : acc[0], k1 = hi16 ? acc[3] : acc[1];
  k0 += __shfl_xor_sync(kFull, s0, 16);
  k1 += __shfl_xor_sync(kFull, s1, 16);
  const bool hi8 = lane & 8;
  const float s = hi8 ? k0 : k1;
  float k = hi8 ? k1 : k0;
  k += __shfl_xor_sync(kFull, s, 8);
  k += __shfl_xor_sync(kFull, k, 4);
  k += __shfl_xor_sync(kFull, k, 2);
  k += __shfl_xor_sync(kFull, k, 1);
  return k;
}

// Stage x[beta][col0 .. col0 + 32*nl) for beta < nb into buf[beta][0 .. 32*P)
// (fp16), zero-filling lanes >= nl and batch rows nb..B-1.  Called by warp 0.
__device__ __forceinline__ void stage_x(__half* buf, uint32_t bar, const __half* x, int n, int col0, int nl,
                                        int P, int nb, int B, int lane) {
  const uint32_t bytes = (uint32_t)nl * 64u;
  if (lane == 0) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, bytes * (uint32_t)nb);
  }
  __syncwarp();
  if (lane < nb) bulk_g2s(smem_u32(buf + (size_t)lane * 32 * P), x + (size_t)lane * n + col0, bytes, bar);
  // zero-fill the rest (generic proxy, disjoint from the async writes)
  const int row_h = 32 * P;
  for (int beta = 0; beta < B; ++beta) {
    const int from = beta < nb ? 32 * nl : 0;
    for (int e = from + lane * 8; e < row_h; e += 32 * 8)
      *reinterpret_cast<uint4*>(buf + (size_t)beta * row_h + e) = make_uint4(0, 0, 0, 0);
  }
}

template <int QT>
struct Ring {
  uint4 k[QT];
  uint2 a[QT];
  uint2 z;
};

template <int QT, bool HAS_Z>
__device__ __forceinline__ void ring_load(Ring<QT>& r, bool ok, const KParams& p, int s, int Ls, int rq, int lay,
                                          int grp, int q) {
  if (ok) {
    const uint8_t* bp = p.planes + plane_vec_offset(p.sh, s, Ls, rq, 0, lay);
    const __half* ap = p.alpha + alpha_index(p.sh, rq, 0, grp, 0);
#pragma unroll
    for (int i = 0; i < QT; ++i) {
      if (QT <= 4 || i < q) {
        r.k[i] = ldg_stream_u4(bp + (size_t)i * Ls * 16);
        r.a[i] = ldg_nc_u2(ap + (size_t)i * p.sh.G * 4);
      } else {
        r.k[i] = make_uint4(0, 0, 0, 0);
        r.a[i] = make_uint2(0, 0);
      }
    }
    if (HAS_Z) r.z = ldg_nc_u2(p.offset + offset_index(p.sh, rq, grp, 0));
  } else {
#pragma unroll
    for (int i = 0; i < QT; ++i) {
      r.k[i] = make_uint4(0, 0, 0, 0);
      r.a[i] = make_uint2(0, 0);
    }
    r.z = make_uint2(0, 0);
  }
}

// acc[r] += sum_i alpha_i[r] * (LUT partial of row r, plane i) (+ z[r] * xsum)
template <int QT, bool HAS_Z>
__device__ __forceinline__ void ring_compute(const Ring<QT>& r, uint32_t lc, float xsum, float acc[4], int q) {
#pragma unroll
  for (int i = 0; i < QT; ++i) {
    if (QT <= 4 || i < q) {
      const float2 a01 = h2_to_f2(r.a[i].x), a23 = h2_to_f2(r.a[i].y);
      acc[0] = fmaf(a01.x, lut4(r.k[i].x, lc), acc[0]);
      acc[1] = fmaf(a01.y, lut4(r.k[i].y, lc), acc[1]);
      acc[2] = fmaf(a23.x, lut4(r.k[i].z, lc), acc[2]);
      acc[3] = fmaf(a23.y, lut4(r.k[i].w, lc), acc[3]);
    }
  }
  if (HAS_Z) {
    const float2 z01 = h2_to_f2(r.z.x), z23 = h2_to_f2(r.z.y);
    acc[0] = fmaf(z01.x, xsum, acc[0]);
    acc[1] = fmaf(z01.y, xsum, acc[1]);
    acc[2] = fmaf(z23.x, xsum, acc[2]);
    acc[3] = fmaf(z23.y, xsum, acc[3]);
  }
}

__device__ __forceinline__ void store_out(const KParams& p, size_t idx, float v) {
  if (p.yf) p.yf[idx] = v;
  else p.y[idx] = __float2half_rn(v);
}

// ---------------------------------------------------------------------------
// GEMV, b = 1 (the paper's single-batch case)
// ---------------------------------------------------------------------------
template <int QT, bool HAS_Z, int PD>
__global__ void __launch_bounds__(kThreads, 1) lut_gemv_kernel(const KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);  // warp-uniform for the compiler
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  const long long it0 = p.items * blockIdx.x / gridDim.x;
  const long long it1 = p.items * (blockIdx.x + 1) / gridDim.x;
  if (it0 >= it1) return;

  const SmemMap sm = map_smem(smem);
  __half* xbuf0 = reinterpret_cast<__half*>(sm.misc_p);
  __half* xbuf1 = reinterpret_cast<__half*>(sm.misc_p + 2048);
  const uint32_t bar0 = sm.misc + 4096, bar1 = sm.misc + 4104;
  volatile unsigned* sflag = reinterpret_cast<volatile unsigned*>(sm.misc_p + 4128);
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)(4 * lane + 128) << 8) | (uint32_t)(4 * lane);

  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    const int s0 = (int)(it0 / sh.RQ);
    stage_x(xbuf0, bar0, p.x, sh.n, s0 * kSliceCols, slice_lanes(sh.n, s0), 32, 1, 1, lane);
  }
  __syncthreads();

  int e = 0;
  long long it = it0;
  while (it < it1) {
    const int s = (int)(it / sh.RQ);
    const int rq_a = (int)(it % sh.RQ);
    const int rq_b = (int)min((long long)sh.RQ, (long long)rq_a + (it1 - it));
    const long long itn = it + (rq_b - rq_a);
    const int Ls = slice_lanes(sh.n, s);
    const bool lane_ok = lane < Ls;
    const int grp = lane_ok ? (s * kSliceCols + 32 * lane) / sh.g : 0;

    // 1. start streaming this segment's first row quads (independent of x)
    Ring<QT> ring[PD];
#pragma unroll
    for (int d = 0; d < PD; ++d) {
      const int rq = rq_a + warp + d * kWarps;
      ring_load<QT, HAS_Z>(ring[d], lane_ok && rq < rq_b, p, s, Ls, rq, lane, grp, q);
    }
    // 2. wait for the staged x slice and build the 128 LUTs of the slice
    __half* xb = (e & 1) ? xbuf1 : xbuf0;
    mbar_wait((e & 1) ? bar1 : bar0, (uint32_t)((e >> 1) & 1));
    {
      const int l = lane, j = warp & 3, h = warp >> 2;
      build_table_part(sm.lut + table_offset(l, j), xb + (4 * l + j) * 8, h);
    }
    __syncthreads();
    // 3. stage the next segment's x slice into the other buffer
    if (warp == 0 && itn < it1) {
      const int sn = (int)(itn / sh.RQ);
      stage_x((e & 1) ? xbuf0 : xbuf1, (e & 1) ? bar0 : bar1, p.x, sh.n, sn * kSliceCols,
              slice_lanes(sh.n, sn), 32, 1, 1, lane);
    }
    float xsum = 0.f;
    if (HAS_Z && lane_ok) {
      const uint32_t k255 = 255u * 256u;
      xsum = (lds_f32<0>(sm.lut + table_offset(lane, 0) + k255) + lds_f32<0>(sm.lut + table_offset(lane, 1) + k255)) +
             (lds_f32<0>(sm.lut + table_offset(lane, 2) + k255) + lds_f32<0>(sm.lut + table_offset(lane, 3) + k255));
    }
    // 4. main loop: row quads rq_a + warp + 16 t
    for (int rq0 = rq_a + warp; rq0 < rq_b; rq0 += PD * kWarps) {
#pragma unroll
      for (int d = 0; d < PD; ++d) {
        const int rq = rq0 + d * kWarps;
        if (rq < rq_b) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          ring_compute<QT, HAS_Z>(ring[d], lc, xsum, acc, q);
          const float v = reduce4(acc, lane);
          if ((lane & 7) == 0) p.partial[(size_t)s * sh.m4 + 4 * rq + (lane >> 3)] = v;
          const int rn = rq + PD * kWarps;
          ring_load<QT, HAS_Z>(ring[d], lane_ok && rn < rq_b, p, s, Ls, rn, lane, grp, q);
        }
      }
    }
    __threadfence();
    __syncthreads();
    // 5. arrival counters per 64-quad block; the last arrival sums the slices
    const int blk_a = rq_a / kBlkQuads, blk_b = (rq_b - 1) / kBlkQuads;
    for (int bb = blk_a; bb <= blk_b; bb += 32) {
      if (warp == 0) {
        const int blk = bb + lane;
        unsigned done = 0;
        if (blk <= blk_b) {
          const int lo = max(rq_a, blk * kBlkQuads), hi = min(rq_b, (blk + 1) * kBlkQuads);
          const unsigned cnt = (unsigned)(hi - lo);
          const unsigned need = (unsigned)sh.S * (unsigned)(min(sh.RQ, (blk + 1) * kBlkQuads) - blk * kBlkQuads);
          const unsigned old = atomicAdd(&p.counters[blk], cnt);
          done = (old + cnt == need);
        }
        const unsigned mask = __ballot_sync(kFull, done);
        __threadfence();
        if (lane == 0) *sflag = mask;
      }
      __syncthreads();
      unsigned mask = *sflag;
      while (mask) {
        const int blk = bb + __ffs(mask) - 1;
        mask &= mask - 1;
        const int row = blk * kBlkQuads * 4 + tid;
        if (tid < kBlkQuads * 4 && row < sh.m) {
          float v = 0.f;
          const float* pp = p.partial + row;
          for (int ss = 0; ss < sh.S; ++ss) v += __ldcg(pp + (size_t)ss * sh.m4);
          store_out(p, (size_t)row, v);
        }
        if (tid == 0) p.counters[blk] = 0u;
      }
      __syncthreads();
    }
    it = itn;
    ++e;
  }
}

// ---------------------------------------------------------------------------
// Batched LUT-GEMM, 2 <= b <= 32.  B = 2^bl >= b table banks
// share each key: lane l = (pp = l >> bl, beta = l & (B-1)); a CTA's 128
// tables hold P = 32/B layout lanes x 4 chunks x B batch rows, so a native
// slice is processed as B sub-slices with register accumulators across them.
// ---------------------------------------------------------------------------
template <int QT, bool HAS_Z, int PD>
__global__ void __launch_bounds__(kThreads, 1) lut_gemm_batched_kernel(const KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  const int bl = p.bl, B = 1 << bl, P = 32 >> bl, b = p.b;
  const int beta = lane & (B - 1), pp = lane >> bl;
  const int rbq = kWarps * kQPW;                      // row quads per work item
  const int NRB = (sh.RQ + rbq - 1) / rbq;
  const long long it0 = p.items * blockIdx.x / gridDim.x;
  const long long it1 = p.items * (blockIdx.x + 1) / gridDim.x;
  if (it0 >= it1) return;

  const SmemMap sm = map_smem(smem);
  __half* xbuf0 = reinterpret_cast<__half*>(sm.misc_p);
  __half* xbuf1 = reinterpret_cast<__half*>(sm.misc_p + 2048);
  const uint32_t bar0 = sm.misc + 4096, bar1 = sm.misc + 4104;
  volatile unsigned* sflag = reinterpret_cast<volatile unsigned*>(sm.misc_p + 4128);
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)(4 * lane + 128) << 8) | (uint32_t)(4 * lane);

  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar1, 1);
    fence_mbar_init();
  }
  __syncthreads();
  // staging of sub-slice (s, k): P lanes starting at layout lane k*P
  auto stage = [&](int ebuf, long long itx, int k) {
    const int s = (int)(itx / NRB);
    const int Ls = slice_lanes(sh.n, s);
    const int nl = min(P, Ls - k * P);
    stage_x((ebuf & 1) ? xbuf1 : xbuf0, (ebuf & 1) ? bar1 : bar0, p.x, sh.n, s * kSliceCols + 32 * k * P, nl, P,
            min(b, B), B, lane);
  };
  if (warp == 0) stage(0, it0, 0);
  __syncthreads();

  int e = 0;
  for (long long it = it0; it < it1; ++it) {
    const int s = (int)(it / NRB);
    const int rb = (int)(it % NRB);
    const int Ls = slice_lanes(sh.n, s);
    const int nsub = (Ls + P - 1) / P;
    const int rq_w = rb * rbq + warp * kQPW;           // this warp's first quad
    float acc[kQPW][4];
#pragma unroll
    for (int t = 0; t < kQPW; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;

    for (int k = 0; k < nsub; ++k, ++e) {
      const int lay = k * P + pp;
      const bool lane_ok = lay < Ls;
      const int grp = lane_ok ? (s * kSliceCols + 32 * lay) / sh.g : 0;
      Ring<QT> ring[PD];
#pragma unroll
      for (int d = 0; d < PD; ++d)
        ring_load<QT, HAS_Z>(ring[d], lane_ok && rq_w + d < sh.RQ, p, s, Ls, rq_w + d, lay, grp, q);
      __half* xb = (e & 1) ? xbuf1 : xbuf0;
      mbar_wait((e & 1) ? bar1 : bar0, (uint32_t)((e >> 1) & 1));
      {
        const int l = lane, j = warp & 3, h = warp >> 2;
        const int bt = l & (B - 1), pl = l >> bl;
        build_table_part(sm.lut + table_offset(l, j), xb + (size_t)bt * 32 * P + (4 * pl + j) * 8, h);
      }
      __syncthreads();
      if (warp == 0) {
        if (k + 1 < nsub) stage(e + 1, it, k + 1);
        else if (it + 1 < it1) stage(e + 1, it + 1, 0);
      }
      float xsum = 0.f;
      if (HAS_Z && lane_ok) {
        const uint32_t k255 = 255u * 256u;
        xsum = (lds_f32<0>(sm.lut + table_offset(lane, 0) + k255) + lds_f32<0>(sm.lut + table_offset(lane, 1) + k255)) +
               (lds_f32<0>(sm.lut + table_offset(lane, 2) + k255) + lds_f32<0>(sm.lut + table_offset(lane, 3) + k255));
      }
#pragma unroll
      for (int t = 0; t < kQPW; ++t) {
        const int d = t % PD;
        ring_compute<QT, HAS_Z>(ring[d], lc, xsum, acc[t], q);
        if (t + PD < kQPW)
          ring_load<QT, HAS_Z>(ring[d], lane_ok && rq_w + t + PD < sh.RQ, p, s, Ls, rq_w + t + PD, lay, grp, q);
      }
      __syncthreads();  // LUT is rebuilt next
    }
    // reduce over the P layout lanes that share a batch row (lane bits >= bl)
#pragma unroll
    for (int t = 0; t < kQPW; ++t) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        float v = acc[t][r];
        for (int off = 16; off >= B; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
        acc[t][r] = v;
      }
    }
    if (pp == 0 && beta < b) {
#pragma unroll
      for (int t = 0; t < kQPW; ++t) {
        const int rq = rq_w + t;
        if (rq < sh.RQ) {
          float* dst = p.partial + ((size_t)s * b + beta) * sh.m4 + 4 * rq;
          *reinterpret_cast<float4*>(dst) = make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const unsigned old = atomicAdd(&p.counters[rb], 1u);
      __threadfence();
      *sflag = (old + 1 == (unsigned)sh.S) ? 1u : 0u;
    }
    __syncthreads();
    if (*sflag) {
      const int row0 = rb * rbq * 4;
      const int nrows = min(sh.m, row0 + rbq * 4) - row0;
      for (int idx = tid; idx < nrows * b; idx += kThreads) {
        const int bt = idx / nrows, row = row0 + idx % nrows;
        float v = 0.f;
        const float* pp2 = p.partial + (size_t)bt * sh.m4 + row;
        for (int ss = 0; ss < sh.S; ++ss) v += __ldcg(pp2 + (size_t)ss * b * sh.m4);
        store_out(p, (size_t)bt * sh.m + row, v);
      }
      if (tid == 0) p.counters[rb] = 0u;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static int g_num_sms[64];

static int num_sms() {
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

template <typename K>
static cudaError_t launch(K kernel, int grid, const KParams& p, cudaStream_t st) {
  cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (err != cudaSuccess) return err;
  kernel<<<grid, kThreads, kSmemBytes, st>>>(p);
  return cudaGetLastError();
}

template <int QT, bool HAS_Z>
static cudaError_t launch_gemv_t(const KParams& p, int grid, cudaStream_t st) {
  constexpr int PD = QT <= 1 ? 6 : (QT <= 2 ? 4 : (QT <= 4 ? 3 : 1));
  return launch(lut_gemv_kernel<QT, HAS_Z, PD>, grid, p, st);
}

template <int QT, bool HAS_Z>
static cudaError_t launch_batched_t(const KParams& p, int grid, cudaStream_t st) {
  constexpr int PD = QT <= 2 ? 4 : (QT <= 4 ? 2 : 1);
  return launch(lut_gemm_batched_kernel<QT, HAS_Z, PD>, grid, p, st);
}

template <bool HAS_Z>
static cudaError_t dispatch_q(const KParams& p, int grid, cudaStream_t st, bool batched) {
  switch (p.sh.q) {
    case 1: return batched ? launch_batched_t<1, HAS_Z>(p, grid, st) : launch_gemv_t<1, HAS_Z>(p, grid, st);
    case 2: return batched ? launch_batched_t<2, HAS_Z>(p, grid, st) : launch_gemv_t<2, HAS_Z>(p, grid, st);
    case 3: return batched ? launch_batched_t<3, HAS_Z>(p, grid, st) : launch_gemv_t<3, HAS_Z>(p, grid, st);
    case 4: return batched ? launch_batched_t<4, HAS_Z>(p, grid, st) : launch_gemv_t<4, HAS_Z>(p, grid, st);
    default: return batched ? launch_batched_t<8, HAS_Z>(p, grid, st) : launch_gemv_t<8, HAS_Z>(p, grid, st);
  }
}

size_t counters_bytes(const Shape& sh) {
  const size_t n = (size_t)(sh.RQ + 15) / 16;
  return (n * 4 + 255) / 256 * 256;
}

size_t workspace_bytes(const Shape& sh, int b) {
  return counters_bytes(sh) + (size_t)sh.S * (size_t)b * (size_t)sh.m4 * 4u;
}

cudaError_t run_product(const Shape& sh, const void* planes, const void* alpha, const void* offset,
                        const uint16_t* x, int b, uint16_t* y, float* yf, void* ws, cudaStream_t st) {
  KParams p;
  p.planes = static_cast<const uint8_t*>(planes);
  p.alpha = static_cast<const __half*>(alpha);
  p.offset = static_cast<const __half*>(offset);
  p.x = reinterpret_cast<const __half*>(x);
  p.y = reinterpret_cast<__half*>(y);
  p.yf = yf;
  p.counters = static_cast<unsigned*>(ws);
  p.partial = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + counters_bytes(sh));
  p.sh = sh;
  p.b = b;
  int bl = 0;
  while ((1 << bl) < b) ++bl;
  p.bl = bl;
  const bool batched = b > 1;
  if (!batched) {
    p.items = (long long)sh.S * sh.RQ;
  } else {
    const int rbq = kWarps * kQPW;
    p.items = (long long)sh.S * ((sh.RQ + rbq - 1) / rbq);
  }
  const int grid = (int)std::min<long long>((long long)num_sms(), p.items);
  return offset ? dispatch_q<true>(p, grid, st, batched) : dispatch_q<false>(p, grid, st, batched);
}

}  // namespace lg
