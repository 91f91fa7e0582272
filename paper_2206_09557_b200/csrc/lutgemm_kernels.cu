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
//  * GEMV: one CTA per SM (512 threads, 16 warps), J CTAs per 1024-column LUT
//    slice; mu = 8, fp32 LUT entries, 128 tables x 256 entries = 128 KB of
//    shared memory per slice, stored interleaved so that entry k of the table
//    used by lane l at chunk step j lives at
//        LUT + (j>>1)*64KB + k*256 + (32*(j&1) + l)*4
//    -> every lookup instruction of a warp hits 32 distinct banks whatever the
//    keys are (bank = lane), and key -> address is ONE byte permute (PRMT)
//    because the LUT sits on a 64 KB boundary of the shared window;
//  * the weight is one slice-major record stream (layout.cuh) read with
//    128-bit loads (L1::no_allocate) through running pointers in a ring of
//    PD + 1 register buffers (loads issued before the lookups of the quad they
//    overtake), no predicates in the steady state;
//  * the activation slice is staged into shared memory by the bulk-copy
//    (TMA) engine after the programmatic-dependent-launch wait;
//  * lookups summed and scaled with packed f32x2 adds/FMAs (FADD2/FFMA2),
//    two rows per instruction;
//  * per-row partials reduced across lanes by a 6-shuffle transpose-reduce and
//    written to an fp32 split-K workspace; the cross-slice sum runs in the same
//    kernel (arrival-ordered, fixed slice order: deterministic);
//  * batched (2 <= b <= 32): vector table slots of V batch rows read with
//    LDS.128 / LDS.64 (see the batched section).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "layout.cuh"
#include "lutgemm_internal.h"
#include "ptx.cuh"

namespace lg {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMiscBytes = 8192;       // x double buffer (2 x 2 KB) + mbarriers + flags
constexpr int kSmemBytes = 3 * 65536;  // LUT (128 KB) on a 64 KB boundary + misc, for any base
constexpr unsigned kFull = 0xffffffffu;
constexpr int kFusedMaxJ = 256;        // max CTAs per slice in the fused-reduction mode

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
// with L over x0..x3 and H over x4..x7: one add per entry (Eq. 2's C_build).
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

// Lookup of key byte J of word w: PRMT places the byte in bits 8..15 next to
// the lane constant lc = LUT[31:16] | (4l+128) << 8 | 4l.
template <int J>
__device__ __forceinline__ float lut1(uint32_t w, uint32_t lc) {
  constexpr uint32_t kSel = ((J & 1) ? 0x7605u : 0x7604u) | ((uint32_t)J << 4);
  return lds_f32<(J >> 1) * 65536>(prmt<kSel>(w, lc));
}

// sum over the 4 keys of word wa (row a) and of word wb (row b), as the pair (a, b)
__device__ __forceinline__ f32x2 lut4x2(uint32_t wa, uint32_t wb, uint32_t lc) {
  const f32x2 p0 = pack2(lut1<0>(wa, lc), lut1<0>(wb, lc));
  const f32x2 p1 = pack2(lut1<1>(wa, lc), lut1<1>(wb, lc));
  const f32x2 p2 = pack2(lut1<2>(wa, lc), lut1<2>(wb, lc));
  const f32x2 p3 = pack2(lut1<3>(wa, lc), lut1<3>(wb, lc));
  return add2(add2(p0, p1), add2(p2, p3));
}

// Transpose-reduce of the 4 per-lane row partials (pairs (0,1), (2,3)) over
// the 32 lanes; returns the full sum of row (lane >> 3) & 3 (valid in lanes
// 0, 8, 16, 24).
__device__ __forceinline__ float reduce4(f32x2 a01, f32x2 a23, int lane) {
  const bool hi16 = lane & 16;
  const f32x2 send = hi16 ? a01 : a23;
  f32x2 keep = hi16 ? a23 : a01;
  const float2 sv = unpack2(send);
  keep = add2(keep, pack2(__shfl_xor_sync(kFull, sv.x, 16), __shfl_xor_sync(kFull, sv.y, 16)));
  const float2 kv = unpack2(keep);
  const bool hi8 = lane & 8;
  const float s = hi8 ? kv.x : kv.y;
  float k = hi8 ? kv.y : kv.x;
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

// One row quad's operands in registers: keys of q planes (4 rows each), the
// lane's group scales (4 rows x q planes, fp16) and bias z (4 rows, fp16).
template <int QT>
struct Ring {
  uint4 k[QT];
  uint2 a[QT];
  uint2 z;
};

// Per-segment addressing of a lane's fields in the three slice regions.
struct LaneAddr {
  const uint8_t* kp;  // lane's key bytes of row quad 0, plane 0
  const uint8_t* ap;  // lane's alpha of row quad 0, plane 0
  const uint8_t* zp;  // lane's z of row quad 0
  uint32_t KB, AB, ZB;  // per-row-quad strides of the regions
  uint32_t kstride;     // bytes between planes of the key block (Ls * 16)
};

__device__ __forceinline__ LaneAddr lane_addr(const Shape& sh, const uint8_t* data, int s, int Ls, int lay) {
  LaneAddr a;
  const int k = lane_group(sh, lay);
  a.kp = data + key_at(sh, s, Ls, 0, 0, lay, 0);
  a.ap = data + alpha_at(sh, s, Ls, 0, 0, k, 0);
  a.zp = data + z_at(sh, s, Ls, 0, k, 0);
  a.KB = keys_bytes(sh, Ls);
  a.AB = alpha_bytes(sh, Ls);
  a.ZB = z_bytes(sh, Ls);
  a.kstride = (uint32_t)Ls * 16u;
  return a;
}

// (acc01, acc23) = sum_i alpha_i[r] * (LUT partial of row r, plane i) (+ z[r] * xsum);
// compact format: (sum_i 2^(i-1) partial_i) * s
template <int QT, int ZM>
__device__ __forceinline__ void ring_compute(const Ring<QT>& r, uint32_t lc, float xsum, f32x2& acc01, f32x2& acc23,
                                             int q) {
  constexpr bool HAS_Z = ZM != 0, CMP = ZM == 2;
  if (CMP) {  // exact power-of-two plane weights, then one multiply by s (App. C)
    f32x2 p01 = 0ull, p23 = 0ull;
#pragma unroll
    for (int i = 0; i < QT; ++i) {
      if (QT <= 4 || i < q) {
        const float w2 = (float)(1 << i) * 0.5f;
        const f32x2 ww = pack2(w2, w2);
        p01 = fma2(ww, lut4x2(r.k[i].x, r.k[i].y, lc), p01);
        p23 = fma2(ww, lut4x2(r.k[i].z, r.k[i].w, lc), p23);
      }
    }
    acc01 = mul2(h2_to_f32x2(r.a[0].x), p01);
    acc23 = mul2(h2_to_f32x2(r.a[0].y), p23);
  } else {
#pragma unroll
    for (int i = 0; i < QT; ++i) {
      if (QT <= 4 || i < q) {
        const f32x2 a01 = h2_to_f32x2(r.a[i].x), a23 = h2_to_f32x2(r.a[i].y);
        const f32x2 s01 = lut4x2(r.k[i].x, r.k[i].y, lc);
        const f32x2 s23 = lut4x2(r.k[i].z, r.k[i].w, lc);
        acc01 = i == 0 ? mul2(a01, s01) : fma2(a01, s01, acc01);
        acc23 = i == 0 ? mul2(a23, s23) : fma2(a23, s23, acc23);
      }
    }
  }
  if (HAS_Z) {
    const f32x2 xs = pack2(xsum, xsum);
    acc01 = fma2(h2_to_f32x2(r.z.x), xs, acc01);
    acc23 = fma2(h2_to_f32x2(r.z.y), xs, acc23);
  }
}

// sum of x over the lane's 32 columns = sum_j T_{4l+j}[255]
__device__ __forceinline__ float lane_xsum(uint32_t lut, int lane) {
  const uint32_t k255 = 255u * 256u;
  return (lds_f32<0>(lut + table_offset(lane, 0) + k255) + lds_f32<0>(lut + table_offset(lane, 1) + k255)) +
         (lds_f32<0>(lut + table_offset(lane, 2) + k255) + lds_f32<0>(lut + table_offset(lane, 3) + k255));
}

// ---------------------------------------------------------------------------
// GEMV, b = 1 (the paper's single-batch case)
//
// Work distribution.  Fused mode (p.fused_J = J > 0, grid S*J <= #SMs): CTA c
// owns slice c / J and row-quad group c % J; the cross-slice reduction runs in
// the kernel (arrival-ordered, below).  Otherwise the S*RQ (slice, row-quad)
// items are split into equal contiguous ranges, one per CTA (a range spans at
// most a few slices), and lut_reduce_kernel follows.  Inside a segment the 16
// warps take row quads rq_a + warp + 16 t round-robin.
// ---------------------------------------------------------------------------
template <int QT, int ZM, int PD>
__global__ void __launch_bounds__(kThreads, 1) lut_gemv_kernel(const KParams p) {
  constexpr bool HAS_Z = ZM != 0, CMP = ZM == 2;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);  // warp-uniform for the compiler
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  const int J = p.fused_J;
  long long it0, it1;
  if (J > 0) {
    const int fs = blockIdx.x / J, fj = blockIdx.x % J;
    it0 = (long long)fs * sh.RQ + (long long)sh.RQ * fj / J;
    it1 = (long long)fs * sh.RQ + (long long)sh.RQ * (fj + 1) / J;
  } else {
    it0 = p.items * blockIdx.x / gridDim.x;
    it1 = p.items * (blockIdx.x + 1) / gridDim.x;
  }
  unsigned long long* trace = (p.trace && tid == 0) ? p.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
  if (trace) {
    trace[0] = globaltimer_ns();
    trace[7] = smid();
  }
  if (it0 >= it1 && J == 0) return;
  // fused mode: the next kernel may launch at once -- its CTAs take SMs as this
  // grid's CTAs exit and stream their first weights before their own PDL wait
  if (J > 0) pdl_launch_dependents();

  const SmemMap sm = map_smem(smem);
  __half* xbuf0 = reinterpret_cast<__half*>(sm.misc_p);
  __half* xbuf1 = reinterpret_cast<__half*>(sm.misc_p + 2048);
  const uint32_t bar0 = sm.misc + 4096, bar1 = sm.misc + 4104;
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)(4 * lane + 128) << 8) | (uint32_t)(4 * lane);
  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar1, 1);
    fence_mbar_init();
  }
  __syncthreads();

  constexpr int NB = PD + 1;  // ring of quad buffers: the load of quad t + PD is issued before quad t is computed
  int e = 0;
  long long it = it0;
  while (it < it1) {
    const int s = (int)(it / sh.RQ);
    const int rq_a = (int)(it % sh.RQ);
    const int rq_b = (int)min((long long)sh.RQ, (long long)rq_a + (it1 - it));
    const long long itn = it + (rq_b - rq_a);
    const int Ls = slice_lanes(sh.n, s);
    const bool lane_ok = lane < Ls;
    const LaneAddr la = lane_addr(sh, p.data, s, Ls, lane_ok ? lane : 0);
    // this warp's row quads in the segment: rq_a + warp + 16 t, t < nt
    const int nt = rq_a + warp < rq_b ? (rq_b - (rq_a + warp) + kWarps - 1) / kWarps : 0;
    // The warp's next quad to load is at (lk, lal, lz); each load advances them
    // by 16 quads unless it was the warp's last, so a load never leaves the
    // warp's range (quads past the end re-read the last one and are not
    // computed) and needs no predicate or zero-fill: the steady-state loop has
    // no branch.  Tail-slice lanes (lane >= Ls) read lane 0's words and are
    // zeroed before the reduction.
    const uint8_t* lk = la.kp + (size_t)(rq_a + warp) * la.KB;
    const uint8_t* lal = la.ap + (size_t)(rq_a + warp) * la.AB;
    const uint8_t* lz = la.zp + (size_t)(rq_a + warp) * la.ZB;
    int tl = 0;
    Ring<QT> buf[NB];
    auto load_quad = [&](Ring<QT>& b) {
      if (nt == 0) return;  // a warp without quads in the segment loads nothing
#pragma unroll
      for (int i = 0; i < QT; ++i) {
        if (QT <= 4 || i < q) {
          b.k[i] = ldg_stream_u4(lk + i * la.kstride);
          if (!CMP || i == 0) b.a[i] = ldg_nc_u2(lal + 8 * i);
        }
      }
      if (HAS_Z) b.z = ldg_nc_u2(lz);
      if (++tl < nt) {
        lk += (size_t)kWarps * la.KB;
        lal += (size_t)kWarps * la.AB;
        if (HAS_Z) lz += (size_t)kWarps * la.ZB;
      }
    };

    // 1. fused mode, first segment: the first PD quads of every warp (weights
    //    only: legal before the PDL wait), then the wait; x (written by the
    //    preceding kernel) is staged by the bulk-copy engine right after it
    if (e == 0) {
      if (J > 0) {
#pragma unroll
        for (int d = 0; d < PD; ++d) load_quad(buf[d]);
      }
      pdl_wait();
      if (trace) trace[5] = globaltimer_ns();
      if (warp == 0) stage_x(xbuf0, bar0, p.x, sh.n, s * kSliceCols, Ls, 32, 1, 1, lane);
    }
    if (e > 0 || J == 0) {
#pragma unroll
      for (int d = 0; d < PD; ++d) load_quad(buf[d]);
    }
    if (e == 0) __syncthreads();  // the zero-fill of the x buffer is visible
    // 2. wait for the staged x slice and build the 128 LUTs of the slice
    __half* xb = (e & 1) ? xbuf1 : xbuf0;
    mbar_wait((e & 1) ? bar1 : bar0, (uint32_t)((e >> 1) & 1));
    if (trace && e == 0) trace[1] = globaltimer_ns();
    {
      const int l = lane, j = warp & 3, h = warp >> 2;
      build_table_part(sm.lut + table_offset(l, j), xb + (4 * l + j) * 8, h);
    }
    __syncthreads();
    if (trace && e == 0) trace[2] = globaltimer_ns();
    // 3. stage the next segment's x slice into the other buffer
    if (warp == 0 && itn < it1) {
      const int sn = (int)(itn / sh.RQ);
      stage_x((e & 1) ? xbuf0 : xbuf1, (e & 1) ? bar0 : bar1, p.x, sh.n, sn * kSliceCols,
              slice_lanes(sh.n, sn), 32, 1, 1, lane);
    }
    const float xsum = (HAS_Z && lane_ok) ? lane_xsum(sm.lut, lane) : 0.f;
    // 4. main loop: per quad and plane 16 PRMT + 16 LDS + 6 FADD2 + 2 FFMA2, then
    //    a 6-shuffle transpose-reduce and one store per row of the slice partial
    float* pw = p.partial + (size_t)s * sh.m4 + 4 * (rq_a + warp) + (lane >> 3);  // this warp's next partial
    auto quad = [&](const Ring<QT>& b) {
      f32x2 acc01, acc23;
      ring_compute<QT, ZM>(b, lc, xsum, acc01, acc23, q);
      if (Ls < kLanesPerSlice && !lane_ok) acc01 = acc23 = 0ull;
      const float v = reduce4(acc01, acc23, lane);
      if ((lane & 7) == 0) *pw = v;
      pw += 4 * kWarps;
    };
    int t0 = 0;
    for (; t0 + NB <= nt; t0 += NB) {
#pragma unroll
      for (int d = 0; d < NB; ++d) {
        load_quad(buf[(d + PD) % NB]);
        quad(buf[d]);
      }
    }
#pragma unroll
    for (int d = 0; d < NB - 1; ++d)
      if (t0 + d < nt) quad(buf[d]);
    if (trace && e == 0) trace[3] = globaltimer_ns();  // warp 0's loop end
    __syncthreads();  // the LUT and x buffer are reused by the next segment
    if (trace) trace[e == 0 ? 4 : 6] = globaltimer_ns();  // all warps done
    it = itn;
    ++e;
  }
  if (trace) trace[7] |= (unsigned long long)e << 32;  // segments processed
  if (J > 0) {
    // Fused cross-slice reduction, arrival-ordered: the S CTAs of row-quad
    // group fj count in with one acq_rel atomic; the first S - R to arrive exit
    // at once (their SMs go to the next kernel), the last R wait for the group
    // and each sums 1/R of its rows over the S slices in slice order
    // (deterministic, R11).  R = p.reducers (1 <= R <= S).
    __shared__ unsigned s_k;
    const int fj = blockIdx.x % J;
    const int R = max(1, min(p.reducers, sh.S));
    unsigned* arrive = p.counters + fj;
    unsigned* depart = p.counters + kFusedMaxJ + fj;
    __syncthreads();  // all partial stores of this CTA are issued
    if (tid == 0) {
      // release: the CTA's partial stores (ordered before by the barrier) are
      // visible to whoever acquires the count; acquire: the last arriver sees all
      s_k = atom_add_acq_rel_u32(arrive, 1u);
    }
    __syncthreads();
    const int k = (int)s_k;
    if (k < sh.S - R) return;
    if (tid == 0 && k != sh.S - 1) {
      while (ld_acquire_u32(arrive) < (unsigned)sh.S) __nanosleep(32);
    }
    __syncthreads();
    if (trace) trace[5] = globaltimer_ns();  // (re-used) the group is complete
    const int ri = k - (sh.S - R);
    const int g0 = (int)((long long)sh.RQ * fj / J), g1 = (int)((long long)sh.RQ * (fj + 1) / J);
    const int r0 = 4 * (g0 + (int)((long long)(g1 - g0) * ri / R));
    const int r1 = min(sh.m, 4 * (g0 + (int)((long long)(g1 - g0) * (ri + 1) / R)));
    for (int r = r0 + tid; r < r1; r += kThreads) {
      float v = 0.f;
      const float* pp = p.partial + r;
      for (int ss0 = 0; ss0 < sh.S; ss0 += 16) {  // up to 16 slices per L2 round trip
        float t[16];
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) t[kk] = (ss0 + kk < sh.S) ? __ldcg(pp + (size_t)(ss0 + kk) * sh.m4) : 0.f;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          if (ss0 + kk < sh.S) v += t[kk];
      }
      if (p.yf) p.yf[r] = v;
      else p.y[r] = __float2half_rn(v);
    }
    __syncthreads();
    if (tid == 0 && atomicAdd(depart, 1u) == (unsigned)R - 1) {  // the last reducer resets the pair
      *arrive = 0u;
      *depart = 0u;
    }
    if (trace) trace[6] = globaltimer_ns();  // reduction share done
    return;
  }
  pdl_launch_dependents();  // the reduction kernel may now be scheduled
}

// ---------------------------------------------------------------------------
// Batched LUT-GEMM, 2 <= b <= 32 ("diminishing performance gains
// as the batch size increases ... memory bandwidth between core and LUTs in
// the shared memory").  The LUT bytes grow x b and the shared-memory crossbar
// (128 B/clk/SM) becomes the roof, so every lookup moves a VECTOR of V batch
// rows: one table slot holds T[key] for V consecutive activation rows, one PRMT
// forms the address and one LDS.128 (V = 4) or LDS.64 (V = 2, b = 2) returns
// V lookups.  A 128 KB LUT holds 128 fp32 per key: C chunks x b_pad rows with
// C * b_pad = 128, so a native slice is processed as sub-slices of NW layout
// lanes (NW * 32 columns), each a LUT rebuild, with register accumulators
// across sub-slices and across the spi slices of a work item.
//
// Lanes: LR = 32 / V lanes form one LDS phase (8 lanes x 16 B or 16 x 8 B =
// 128 B); lane = rg * LR + wv, wv = w * NV + v: row group rg (4 / V rows of the
// row quad), layout lane w of the sub-slice, batch vector v (rows vV..vV+V-1).
// Slot of (chunk 4w + J, vector v) for key k:
//     LUT + (J >> 1) * 64 KB + k * 256 + (LR * (J & 1) + wv) * 4V
// The LR lanes of a phase have distinct wv, hence distinct 4V-byte bank groups
// whatever their keys: conflict-free by construction, and key -> address is
// still one PRMT (the key byte lands in bits 8..15 next to a lane constant).
// ---------------------------------------------------------------------------

// V lookups of key byte J of word w, as V/2 packed f32x2
template <int V, int J>
__device__ __forceinline__ void vlut(uint32_t w, uint32_t lc, f32x2 (&t)[V / 2]) {
  constexpr uint32_t kSel = ((J & 1) ? 0x7605u : 0x7604u) | ((uint32_t)J << 4);
  const uint32_t a = prmt<kSel>(w, lc);
  if constexpr (V == 4) lds_b64x2<(J >> 1) * 65536>(a, t[0], t[1]);
  else t[0] = lds_b64<(J >> 1) * 65536>(a);
}

// sum of the 4 chunk lookups of word w (32 columns) for the lane's V batch rows
template <int V>
__device__ __forceinline__ void vword(uint32_t w, uint32_t lc, f32x2 (&s)[V / 2]) {
  f32x2 t0[V / 2], t1[V / 2], t2[V / 2], t3[V / 2];
  vlut<V, 0>(w, lc, t0);
  vlut<V, 1>(w, lc, t1);
  vlut<V, 2>(w, lc, t2);
  vlut<V, 3>(w, lc, t3);
#pragma unroll
  for (int p = 0; p < V / 2; ++p) s[p] = add2(add2(t0[p], t1[p]), add2(t2[p], t3[p]));
}

// x tile of a sub-slice in shared memory: 128 16-byte cells (8 columns of one
// activation row each); cell of (column chunk c = 4w + J4, row bt = vV + u) is
//     (J4 * V + u) * LR + w * NV + v
// so the 8 builder lanes of one LDS.128 phase (same J4 and u, distinct (w, v))
// read 8 distinct cells of one 128-byte line: conflict-free.
template <int V>
__device__ __forceinline__ int xcell(int c, int bt, int NV) {
  constexpr int LR = 32 / V;
  return ((c & 3) * V + bt % V) * LR + (c >> 2) * NV + bt / V;
}

// Build the sub-slice LUT: slot (region R, key k, slot s) holds
// T_c[k] for rows vV..vV+V-1 of chunk c = 4w + 2R + s / LR, with (w, v) from
// wv = s % LR.  T[k] = H(k >> 4) + (+-x0 +- x1) + (+-x2 +- x3): with
// A1 = x0 - x1, A3 = x0 + x1 the low pair takes -A3, A1, -A1, A3 (likewise B
// over x2, x3), so each entry costs one packed add after 4 adds per (h, pair).
template <int V, int NTH>
__device__ __forceinline__ void build_vtables(uint32_t lut, const __half* tile, int NV, int tid) {
  constexpr int LR = 32 / V, NP = V / 2;
  constexpr int SPR = 2 * LR;                      // slots per region and key
  constexpr int TPR = NTH / 2;                     // threads per region
  constexpr int HPT = 16 * SPR / TPR;              // high nibbles per thread
  const int R = tid / TPR, rem = tid % TPR;
  const int s = rem % SPR, h0 = rem / SPR;
  const int Jp = s / LR, wv = s % LR, w = wv / NV, v = wv % NV;
  const int c = 4 * w + 2 * R + Jp;
  f32x2 A1[NP], A3[NP], B1[NP], B3[NP], X4[NP], X5[NP], X6[NP], X7[NP];
#pragma unroll
  for (int pp = 0; pp < NP; ++pp) {
    float x[2][8];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const uint4 raw = *reinterpret_cast<const uint4*>(tile + 8 * xcell<V>(c, v * V + 2 * pp + e, NV));
      const float2 a = h2_to_f2(raw.x), b = h2_to_f2(raw.y), cc = h2_to_f2(raw.z), d = h2_to_f2(raw.w);
      x[e][0] = a.x; x[e][1] = a.y; x[e][2] = b.x; x[e][3] = b.y;
      x[e][4] = cc.x; x[e][5] = cc.y; x[e][6] = d.x; x[e][7] = d.y;
    }
    const f32x2 x0 = pack2(x[0][0], x[1][0]), x1 = pack2(x[0][1], x[1][1]);
    const f32x2 x2 = pack2(x[0][2], x[1][2]), x3 = pack2(x[0][3], x[1][3]);
    A1[pp] = sub2(x0, x1); A3[pp] = add2(x0, x1);
    B1[pp] = sub2(x2, x3); B3[pp] = add2(x2, x3);
    X4[pp] = pack2(x[0][4], x[1][4]); X5[pp] = pack2(x[0][5], x[1][5]);
    X6[pp] = pack2(x[0][6], x[1][6]); X7[pp] = pack2(x[0][7], x[1][7]);
  }
#pragma unroll
  for (int hh = 0; hh < HPT; ++hh) {
    const int h = h0 + hh * (16 / HPT);  // key bits 4..7
    const float g4 = (h & 1) ? 1.f : -1.f, g5 = (h & 2) ? 1.f : -1.f;
    const float g6 = (h & 4) ? 1.f : -1.f, g7 = (h & 8) ? 1.f : -1.f;
    f32x2 HA[4][NP];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) {
      const f32x2 H = fma2(pack2(g4, g4), X4[pp], fma2(pack2(g5, g5), X5[pp],
                           fma2(pack2(g6, g6), X6[pp], mul2(pack2(g7, g7), X7[pp]))));
      HA[0][pp] = sub2(H, A3[pp]);
      HA[1][pp] = add2(H, A1[pp]);
      HA[2][pp] = sub2(H, A1[pp]);
      HA[3][pp] = add2(H, A3[pp]);
    }
    const uint32_t base = lut + (uint32_t)R * 65536u + (uint32_t)(16 * h) * 256u + (uint32_t)s * (4u * V);
#pragma unroll
    for (int lo = 0; lo < 16; ++lo) {
      f32x2 e[NP];
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        const int k2 = lo >> 2;
        const f32x2 ha = HA[lo & 3][pp];
        e[pp] = k2 == 0 ? sub2(ha, B3[pp]) : (k2 == 1 ? add2(ha, B1[pp]) : (k2 == 2 ? sub2(ha, B1[pp]) : add2(ha, B3[pp])));
      }
      if constexpr (V == 4) sts_b64x2(base + lo * 256u, e[0], e[1]);
      else sts_b64(base + lo * 256u, e[0]);
    }
  }
}

// The lane's running pointers into the three regions of one slice: plane i's
// key words of the lane's next quad at kq + i * kstride, its scales at
// aq + 8 i, its z at zq; each advances by V quads per step.
struct VPtr {
  const uint8_t *kq, *aq, *zq;
  uint32_t KB, AB, ZB, kstride;  // per-step strides (V quads) and the plane stride
};

template <int QT, int ZM>
__device__ __forceinline__ void vring_load(Ring<QT>& r, bool ok, VPtr& pt, int q) {
  constexpr bool HAS_Z = ZM != 0, CMP = ZM == 2;  // z term; compact scales (alpha_i = 2^(i-1) s)
#pragma unroll
  for (int i = 0; i < QT; ++i) {
    if (QT <= 4 || i < q) {
      if (ok) {
        r.k[i] = ldg_stream_u4(pt.kq + i * pt.kstride);
        r.a[i] = (!CMP || i == 0) ? ldg_nc_u2(pt.aq + 8 * i) : make_uint2(0, 0);
      } else {
        r.k[i] = make_uint4(0, 0, 0, 0);
        r.a[i] = make_uint2(0, 0);
      }
    }
  }
  if (HAS_Z) r.z = ok ? ldg_nc_u2(pt.zq) : make_uint2(0, 0);
  pt.kq += pt.KB;
  pt.aq += pt.AB;
  if (HAS_Z) pt.zq += pt.ZB;
}

// acc[rho][p] (+)= sum_i alpha_i[rho] * (word lookups of row rho, plane i) + z[rho] * xsum, rho < 4
template <int V, int QT, int ZM>
__device__ __forceinline__ void vring_compute(const Ring<QT>& r, uint32_t lc, const f32x2 (&xs)[V / 2],
                                              f32x2 (&acc)[4][V / 2], int q) {
  constexpr bool HAS_Z = ZM != 0, CMP = ZM == 2;  // z term; compact scales (alpha_i = 2^(i-1) s)
  constexpr int NP = V / 2;
  f32x2 P[4][NP];  // compact: sum_i 2^(i-1) (plane i lookups), scaled by s after the planes
#pragma unroll
  for (int i = 0; i < QT; ++i) {
    if (QT <= 4 || i < q) {
      const uint32_t kw[4] = {r.k[i].x, r.k[i].y, r.k[i].z, r.k[i].w};
      const float2 a01 = h2_to_f2(r.a[i].x), a23 = h2_to_f2(r.a[i].y);
      const float w2 = (float)(1 << i) * 0.5f;
      const float al[4] = {CMP ? w2 : a01.x, CMP ? w2 : a01.y, CMP ? w2 : a23.x, CMP ? w2 : a23.y};
      // all 16 lookups of the plane are issued before the first add (ILP over
      // the LDS latency), then summed per row and scaled
      f32x2 t[4][4][NP];
#pragma unroll
      for (int rho = 0; rho < 4; ++rho) {
        vlut<V, 0>(kw[rho], lc, t[rho][0]);
        vlut<V, 1>(kw[rho], lc, t[rho][1]);
        vlut<V, 2>(kw[rho], lc, t[rho][2]);
        vlut<V, 3>(kw[rho], lc, t[rho][3]);
      }
#pragma unroll
      for (int rho = 0; rho < 4; ++rho) {
        const f32x2 aa = pack2(al[rho], al[rho]);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const f32x2 s = add2(add2(t[rho][0][p], t[rho][1][p]), add2(t[rho][2][p], t[rho][3][p]));
          if (!CMP) acc[rho][p] = fma2(aa, s, acc[rho][p]);
          else P[rho][p] = i == 0 ? mul2(aa, s) : fma2(aa, s, P[rho][p]);
        }
      }
    }
  }
  if (CMP) {
    const float2 s01 = h2_to_f2(r.a[0].x), s23 = h2_to_f2(r.a[0].y);
    const float sv[4] = {s01.x, s01.y, s23.x, s23.y};
#pragma unroll
    for (int rho = 0; rho < 4; ++rho)
#pragma unroll
      for (int p = 0; p < NP; ++p) acc[rho][p] = fma2(pack2(sv[rho], sv[rho]), P[rho][p], acc[rho][p]);
  }
  if (HAS_Z) {
    const float2 z01 = h2_to_f2(r.z.x), z23 = h2_to_f2(r.z.y);
    const float zv[4] = {z01.x, z01.y, z23.x, z23.y};
#pragma unroll
    for (int rho = 0; rho < 4; ++rho) {
      const f32x2 zz = pack2(zv[rho], zv[rho]);
#pragma unroll
      for (int p = 0; p < NP; ++p) acc[rho][p] = fma2(zz, xs[p], acc[rho][p]);
    }
  }
}

// A step of the work loop: sub-slice k of slice s of work item it.
struct VStep {
  int it, s, k;
  int s_end;  // end of the item's slice range
  int nsub;   // sub-slices of slice s
};

// Lanes: lane = qi * LR + wv: quad qi of each group of V consecutive quads
// (all 4 rows of it), wv = w * NV + v as above.  A warp owns QPW consecutive
// quads of the work item's row block, processed as QPW / V steps.
template <int V, int QT, int ZM, int PD, int QPW, int NTH>
__global__ void __launch_bounds__(NTH, 1) lut_gemm_batched_kernel(const KParams p) {
  constexpr bool HAS_Z = ZM != 0;
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int LR = 32 / V, NP = V / 2, NB = PD + 1, NT = QPW / V;
  static_assert(QPW % V == 0 && NT % NB == 0, "the ring restarts at buffer 0 every sub-slice");
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  const int NV = p.nv, NW = LR / NV, bpad = V * NV, b = p.b, spi = p.spi;
  const int qi = lane / LR, wv = lane % LR, w = wv / NV, v = wv % NV;
  const int rbq = (NTH / 32) * QPW;  // row quads per work item
  const int NRB = (sh.RQ + rbq - 1) / rbq;
  const int it0 = (int)(p.items * blockIdx.x / gridDim.x);
  const int it1 = (int)(p.items * (blockIdx.x + 1) / gridDim.x);
  if (it0 >= it1) return;

  const SmemMap sm = map_smem(smem);
  const __half* xtile0 = reinterpret_cast<const __half*>(sm.misc_p);
  const __half* xtile1 = reinterpret_cast<const __half*>(sm.misc_p + 2048);
  const uint32_t xt0 = sm.misc, xt1 = sm.misc + 2048;
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)((LR + wv) * 4 * V) << 8) | (uint32_t)(wv * 4 * V);
  const int gsh = p.gsh;  // layout lane p's group in the slice = p >> gsh

  auto nsub_of = [&](int s) { return (slice_lanes(sh.n, s) + NW - 1) / NW; };
  auto first_step = [&](int it) {
    VStep st;
    st.it = it;
    st.s = (it / NRB) * spi;
    st.s_end = min(sh.S, st.s + spi);
    st.k = 0;
    st.nsub = nsub_of(st.s);
    return st;
  };
  auto next_step = [&](VStep st) {
    if (++st.k < st.nsub) return st;
    st.k = 0;
    if (++st.s < st.s_end) {
      st.nsub = nsub_of(st.s);
      return st;
    }
    return first_step(st.it + 1);
  };
  // x tile of a step: x[beta][col0 .. col0 + 32 NW) for beta < b_pad (zero for
  // beta >= b and lanes past the slice end), one 16-byte cp.async per thread
  // for the first 128 threads (2 KB), x is L2-resident
  auto load_x = [&](uint32_t dst, const VStep& st) {
    if (tid < 128) {
      const int Ls = slice_lanes(sh.n, st.s);
      const int per_row = 4 * NW;  // 16-byte cells per tile row
      const int bt = tid / per_row, c = tid % per_row;
      const bool ok = bt < b && st.k * NW + c / 4 < Ls;
      const __half* src = ok ? p.x + (size_t)bt * sh.n + st.s * kSliceCols + 32 * st.k * NW + 8 * c : p.x;
      cp_async_16(dst + 16u * (uint32_t)xcell<V>(c, bt, NV), src, ok ? 16u : 0u);
    }
  };
  // the lane's pointers at its quad of the warp's first group (quad rq_w + qi)
  auto lane_ptr = [&](const VStep& st, int rq_w, bool& ok) {
    const int Ls = slice_lanes(sh.n, st.s);
    const int lay = st.k * NW + w;
    ok = lay < Ls;
    const int pl = ok ? lay : 0;
    const int rq = rq_w + qi;
    VPtr pt;
    const uint32_t KB = keys_bytes(sh, Ls), AB = alpha_bytes(sh, Ls), ZB = z_bytes(sh, Ls);
    pt.KB = KB * V;
    pt.AB = AB * V;
    pt.ZB = ZB * V;
    pt.kstride = (uint32_t)Ls * 16u;
    pt.kq = p.data + keys_base(sh, st.s, Ls) + (size_t)rq * KB + pl * 16;
    pt.aq = p.data + alpha_base(sh, st.s, Ls) + (size_t)rq * AB + (uint32_t)(pl >> gsh) * scale_planes(sh) * 8u;
    pt.zq = p.data + z_base(sh, st.s, Ls) + (size_t)rq * ZB + (uint32_t)(pl >> gsh) * 8u;
    return pt;
  };
  Ring<QT> ring[NB];
  VPtr nxt;  // pointers of the next step, positioned after its prologue groups
  bool nxt_ok;
  auto prologue = [&](const VStep& st) {
    const int rq_w = (st.it % NRB) * rbq + warp * QPW;
    nxt = lane_ptr(st, rq_w, nxt_ok);
#pragma unroll
    for (int d = 0; d < PD; ++d) vring_load<QT, ZM>(ring[d], nxt_ok && rq_w + V * d + qi < sh.RQ, nxt, q);
  };

  VStep st = first_step(it0);
  prologue(st);  // weights only: legal before the PDL wait
  pdl_wait();    // x and the workspace belong to the preceding kernel until it completes
  load_x(xt0, st);
  cp_async_wait_all();
  __syncthreads();
  int e = 0;  // steps processed: x tile e & 1

  while (st.it < it1) {
    const int it = st.it;
    const int rq_w = (it % NRB) * rbq + warp * QPW;  // this warp's first quad
    const int nql = sh.RQ - (rq_w + qi);             // quads from the lane's first one to the end
    f32x2 acc[NT][4][NP];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int rho = 0; rho < 4; ++rho)
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) acc[t][rho][pp] = 0ull;
    const int sr = it / NRB;
    while (st.it == it) {  // the slices and sub-slices of this item
      VPtr cur = nxt;
      const bool lane_ok = nxt_ok;
      build_vtables<V, NTH>(sm.lut, (e & 1) ? xtile1 : xtile0, NV, tid);
      __syncthreads();
      const VStep sn = next_step(st);
      if (sn.it < it1) load_x((e & 1) ? xt0 : xt1, sn);  // lands during the lookups
      f32x2 xs[NP];
      if (HAS_Z) vword<V>(0xFFFFFFFFu, lc, xs);  // sum of x over the lane's 32 columns = sum_J T_J[255]
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (t + PD < NT) vring_load<QT, ZM>(ring[(t + PD) % NB], lane_ok && V * (t + PD) < nql, cur, q);
        vring_compute<V, QT, ZM>(ring[t % NB], lc, xs, acc[t], q);
      }
      if (sn.it < it1) prologue(sn);  // next step's first quads fly during the barrier and rebuild
      cp_async_wait_all();
      __syncthreads();  // every warp is done with the LUT; the next x tile is visible
      st = sn;
      ++e;
    }
    // reduce over the NW layout lanes of a quad (lane bits log2(NV) .. log2(LR)-1)
    float* part = p.partial + (size_t)sr * sh.m4 * bpad;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
#pragma unroll
      for (int rho = 0; rho < 4; ++rho) {
        float2 f[NP];
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
          f[pp] = unpack2(acc[t][rho][pp]);
          for (int off = NV; off < LR; off <<= 1) {
            f[pp].x += __shfl_xor_sync(kFull, f[pp].x, off);
            f[pp].y += __shfl_xor_sync(kFull, f[pp].y, off);
          }
        }
        if (w == 0 && V * t < nql) {
          float* dst = part + (size_t)(4 * (rq_w + qi + V * t) + rho) * bpad + v * V;
          if constexpr (V == 4) *reinterpret_cast<float4*>(dst) = make_float4(f[0].x, f[0].y, f[1].x, f[1].y);
          else *reinterpret_cast<float2*>(dst) = f[0];
        }
      }
    }
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// b <= 4 with the GEMV's streaming structure.  With V = 2 (b = 2) or V = 4
// (b = 3, 4) a sub-slice of 1024 / V columns (layout lanes [LR h, LR h + LR) of a
// slice, LR = 32 / V; sub-slice hs = V s + h) holds the LUTs of all V
// activation rows: 32 LR... = 128 KB of V-float vector slots (the batched
// kernel's slot layout with NV = 1), read with one PRMT + LDS.64 / LDS.128 per
// key.  Lane l = qi * LR + w owns quad qi of a group of V consecutive row quads
// and word w; a warp step is one quad group.  Unlike the batched kernel there
// are no accumulators across LUT rebuilds: each quad's 4 rows x V partials are
// reduced over its LR lanes right away (transpose-reduce) and stored as a
// sub-slice partial, so registers go to a PD-deep load ring as in the GEMV; the
// cross-sub-slice sum is the GEMV's fused arrival-ordered reduction (or
// lut_reduce_kernel when the sub-slices outnumber the SMs).
// Partials [SV][b][m4], SV = sub-slices.
// ---------------------------------------------------------------------------

// V = 2: the 4 rows x 2 batch sums of a quad over the 16 lanes sharing qi;
// lane keeps (row (lane >> 2) & 3, batch (lane >> 1) & 1), valid in even lanes
__device__ __forceinline__ void reduce_quad(const f32x2 (&acc)[4][1], int lane, float (&out)[1]) {
  float2 v[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) v[r] = unpack2(acc[r][0]);
  const bool b3 = lane & 8;
  float k0x = b3 ? v[2].x : v[0].x, k0y = b3 ? v[2].y : v[0].y, k1x = b3 ? v[3].x : v[1].x, k1y = b3 ? v[3].y : v[1].y;
  const float s0x = b3 ? v[0].x : v[2].x, s0y = b3 ? v[0].y : v[2].y, s1x = b3 ? v[1].x : v[3].x, s1y = b3 ? v[1].y : v[3].y;
  k0x += __shfl_xor_sync(kFull, s0x, 8);
  k0y += __shfl_xor_sync(kFull, s0y, 8);
  k1x += __shfl_xor_sync(kFull, s1x, 8);
  k1y += __shfl_xor_sync(kFull, s1y, 8);
  const bool b2 = lane & 4;
  float kx = b2 ? k1x : k0x, ky = b2 ? k1y : k0y;
  const float sx = b2 ? k0x : k1x, sy = b2 ? k0y : k1y;
  kx += __shfl_xor_sync(kFull, sx, 4);
  ky += __shfl_xor_sync(kFull, sy, 4);
  const bool b1 = lane & 2;
  float k = b1 ? ky : kx;
  k += __shfl_xor_sync(kFull, b1 ? kx : ky, 2);
  k += __shfl_xor_sync(kFull, k, 1);
  out[0] = k;
}

// V = 4: the 4 rows x 4 batch sums of a quad over the 8 lanes sharing qi; lane
// keeps row 2 (lane >> 2 & 1) + (lane >> 1 & 1), batch pair (lane & 1) (two values)
__device__ __forceinline__ void reduce_quad(const f32x2 (&acc)[4][2], int lane, float (&out)[2]) {
  const bool b2 = lane & 4, b1 = lane & 2, b0 = lane & 1;
  // xor 4: keep rows {0,1} or {2,3} (8 values)
  f32x2 k[2][2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      const f32x2 keep = b2 ? acc[2 + r][p] : acc[r][p], send = b2 ? acc[r][p] : acc[2 + r][p];
      const float2 sv = unpack2(send);
      k[r][p] = add2(keep, pack2(__shfl_xor_sync(kFull, sv.x, 4), __shfl_xor_sync(kFull, sv.y, 4)));
    }
  // xor 2: keep one row of the pair (4 values)
  f32x2 m[2];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const f32x2 keep = b1 ? k[1][p] : k[0][p], send = b1 ? k[0][p] : k[1][p];
    const float2 sv = unpack2(send);
    m[p] = add2(keep, pack2(__shfl_xor_sync(kFull, sv.x, 2), __shfl_xor_sync(kFull, sv.y, 2)));
  }
  // xor 1: keep batch pair (0,1) or (2,3) (2 values)
  const f32x2 keep = b0 ? m[1] : m[0], send = b0 ? m[0] : m[1];
  const float2 sv = unpack2(send);
  const float2 r = unpack2(add2(keep, pack2(__shfl_xor_sync(kFull, sv.x, 1), __shfl_xor_sync(kFull, sv.y, 1))));
  out[0] = r.x;
  out[1] = r.y;
}

template <int V, int QT, int ZM, int PD>
__global__ void __launch_bounds__(kThreads, 1) lut_gemvv_kernel(const KParams p) {
  constexpr bool HAS_Z = ZM != 0, CMP = ZM == 2;
  constexpr int NB = PD + 1, LR = 32 / V, NP = V / 2;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);
  const int qi = lane / LR, w = lane % LR;
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  const int b = p.b;
  const int NG = (sh.RQ + V - 1) / V;  // quad groups
  const int SV = p.s2;                 // sub-slices
  const int J = p.fused_J;
  long long it0, it1;  // items = (sub-slice, quad group)
  if (J > 0) {
    const int fs = blockIdx.x / J, fj = blockIdx.x % J;
    it0 = (long long)fs * NG + (long long)NG * fj / J;
    it1 = (long long)fs * NG + (long long)NG * (fj + 1) / J;
  } else {
    it0 = p.items * blockIdx.x / gridDim.x;
    it1 = p.items * (blockIdx.x + 1) / gridDim.x;
  }
  if (it0 >= it1 && J == 0) return;
  if (J > 0) pdl_launch_dependents();

  const SmemMap sm = map_smem(smem);
  const uint32_t xt0 = sm.misc, xt1 = sm.misc + 2048;
  const __half* xtile0 = reinterpret_cast<const __half*>(sm.misc_p);
  const __half* xtile1 = reinterpret_cast<const __half*>(sm.misc_p + 2048);
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)((LR + w) * 4 * V) << 8) | (uint32_t)(w * 4 * V);
  // x tile of sub-slice hs: rows 0..V-1 of x (zero for rows >= b), 32 LR columns,
  // in the vector-slot cell order (xcell<V>, NV = 1)
  auto load_x = [&](uint32_t dst, int hs) {
    if (tid < 128) {
      const int s = hs / V, h = hs % V;
      const int Lh = min(LR, slice_lanes(sh.n, s) - LR * h);
      const int per_row = 4 * LR;
      const int bt = tid / per_row, c = tid % per_row;
      const bool ok = bt < b && c / 4 < Lh;
      const __half* src = ok ? p.x + (size_t)bt * sh.n + s * kSliceCols + 32 * LR * h + 8 * c : p.x;
      cp_async_16(dst + 16u * (uint32_t)xcell<V>(c, bt, 1), src, ok ? 16u : 0u);
    }
  };

  int e = 0;
  long long it = it0;
  while (it < it1) {
    const int hs = (int)(it / NG);
    const int ga = (int)(it % NG);
    const int gb = (int)min((long long)NG, (long long)ga + (it1 - it));
    const long long itn = it + (gb - ga);
    const int s = hs / V, h = hs % V;
    const int Ls = slice_lanes(sh.n, s);
    const int Lh = min(LR, Ls - LR * h);
    const bool lane_ok = w < Lh;
    const LaneAddr la = lane_addr(sh, p.data, s, Ls, LR * h + (lane_ok ? w : 0));
    // this warp's groups ga + warp + 16 t, t < nt; the lane's quad V group + qi exists for t < ntl
    const int nt = ga + warp < gb ? (gb - (ga + warp) + kWarps - 1) / kWarps : 0;
    const int last_quad = V * (ga + warp + kWarps * (nt - 1)) + qi;
    const int ntl = nt - (nt > 0 && last_quad >= sh.RQ ? 1 : 0);
    const int rq0 = V * (ga + warp) + qi;
    const uint8_t* lk = la.kp + (size_t)rq0 * la.KB;
    const uint8_t* lal = la.ap + (size_t)rq0 * la.AB;
    const uint8_t* lz = la.zp + (size_t)rq0 * la.ZB;
    int tl = 0;
    Ring<QT> buf[NB];
    auto load_group = [&](Ring<QT>& bb) {
      if (ntl <= 0) return;  // nothing valid for this lane: no loads (its first quad is past the range)
#pragma unroll
      for (int i = 0; i < QT; ++i) {
        if (QT <= 4 || i < q) {
          bb.k[i] = ldg_stream_u4(lk + i * la.kstride);
          if (!CMP || i == 0) bb.a[i] = ldg_nc_u2(lal + 8 * i);
        }
      }
      if (HAS_Z) bb.z = ldg_nc_u2(lz);
      if (++tl < ntl) {
        lk += (size_t)(V * kWarps) * la.KB;
        lal += (size_t)(V * kWarps) * la.AB;
        if (HAS_Z) lz += (size_t)(V * kWarps) * la.ZB;
      }
    };
    if (e == 0) {
      if (J > 0) {
#pragma unroll
        for (int d = 0; d < PD; ++d) load_group(buf[d]);
      }
      pdl_wait();
      load_x(xt0, hs);
    }
    if (e > 0 || J == 0) {
#pragma unroll
      for (int d = 0; d < PD; ++d) load_group(buf[d]);
    }
    cp_async_wait_all();
    __syncthreads();  // the x tile is visible
    build_vtables<V, kThreads>(sm.lut, (e & 1) ? xtile1 : xtile0, 1, tid);
    __syncthreads();
    if (itn < it1) load_x((e & 1) ? xt0 : xt1, (int)(itn / NG));  // lands during the lookups
    f32x2 xs[NP];
    if (HAS_Z) vword<V>(0xFFFFFFFFu, lc, xs);  // sum of x (all rows) over the lane's 32 columns
    // the even / all lanes of a quad store (batch, row) sums; partial [hs][beta][4 rq + row]
    float* pw = p.partial + (size_t)hs * b * sh.m4 + 4 * rq0;
    auto group = [&](const Ring<QT>& bb, bool valid) {
      f32x2 acc[4][NP];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) acc[r][pp] = 0ull;
      vring_compute<V, QT, ZM>(bb, lc, xs, acc, q);
      if (!valid || (Lh < LR && !lane_ok))
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) acc[r][pp] = 0ull;
      float out[NP];
      reduce_quad(acc, lane, out);
      if (valid) {
        if constexpr (V == 2) {
          if ((lane & 1) == 0) pw[((lane >> 1) & 1) * sh.m4 + ((lane >> 2) & 3)] = out[0];
        } else {
          const int row = 2 * ((lane >> 2) & 1) + ((lane >> 1) & 1), beta = 2 * (lane & 1);
          if (beta < b) pw[beta * sh.m4 + row] = out[0];
          if (beta + 1 < b) pw[(beta + 1) * sh.m4 + row] = out[1];
        }
      }
      pw += 4 * V * kWarps;
    };
    int t0 = 0;
    for (; t0 + NB <= nt; t0 += NB) {
#pragma unroll
      for (int d = 0; d < NB; ++d) {
        load_group(buf[(d + PD) % NB]);
        group(buf[d], t0 + d < ntl);
      }
    }
#pragma unroll
    for (int d = 0; d < NB - 1; ++d)
      if (t0 + d < nt) group(buf[d], t0 + d < ntl);
    __syncthreads();  // the LUT and x tile are reused by the next segment
    it = itn;
    ++e;
  }
  if (J > 0) {  // fused arrival-ordered reduction over the SV sub-slices (as in lut_gemv_kernel)
    __shared__ unsigned s_k;
    const int fj = blockIdx.x % J;
    const int R = max(1, min(p.reducers, SV));
    unsigned* arrive = p.counters + fj;
    unsigned* depart = p.counters + kFusedMaxJ + fj;
    __syncthreads();
    if (tid == 0) s_k = atom_add_acq_rel_u32(arrive, 1u);
    __syncthreads();
    const int k = (int)s_k;
    if (k < SV - R) return;
    if (tid == 0 && k != SV - 1) {
      while (ld_acquire_u32(arrive) < (unsigned)SV) __nanosleep(32);
    }
    __syncthreads();
    const int ri = k - (SV - R);
    const int g0 = V * (int)((long long)NG * fj / J), g1 = min(sh.RQ, V * (int)((long long)NG * (fj + 1) / J));
    const int r0 = 4 * (g0 + (int)((long long)(g1 - g0) * ri / R));
    const int r1 = min(sh.m, 4 * (g0 + (int)((long long)(g1 - g0) * (ri + 1) / R)));
    const int nr = max(0, r1 - r0);
    for (int idx = tid; idx < b * nr; idx += kThreads) {
      const int beta = idx / nr, r = r0 + idx % nr;
      float v = 0.f;
      const float* pp = p.partial + (size_t)beta * sh.m4 + r;
      for (int ss0 = 0; ss0 < SV; ss0 += 16) {
        float t[16];
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          t[kk] = (ss0 + kk < SV) ? __ldcg(pp + (size_t)(ss0 + kk) * b * sh.m4) : 0.f;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          if (ss0 + kk < SV) v += t[kk];
      }
      if (p.yf) p.yf[(size_t)beta * sh.m + r] = v;
      else p.y[(size_t)beta * sh.m + r] = __float2half_rn(v);
    }
    __syncthreads();
    if (tid == 0 && atomicAdd(depart, 1u) == (unsigned)R - 1) {
      *arrive = 0u;
      *depart = 0u;
    }
    return;
  }
  pdl_launch_dependents();
}

// Batched cross-slice reduction: Y[beta][r] = sum_{s<S2} partial[s][r][beta]
// in slice order (deterministic, R11), fp16 RNE (or fp32).  A block owns 64
// rows: coalesced reads of the [row][b_pad] partials, transposed in shared
// memory, coalesced writes of Y rows.
__global__ void __launch_bounds__(256) lut_reduce_batched_kernel(const float* __restrict__ partial, int S2, int b,
                                                                 int bpad, int m, int m4, __half* __restrict__ y,
                                                                 float* __restrict__ yf) {
  __shared__ float tile[32][65];
  pdl_launch_dependents();
  pdl_wait();
  const int row0 = blockIdx.x * 64;
  for (int e = threadIdx.x; e < 64 * bpad; e += 256) {
    const int r = e / bpad, beta = e % bpad;
    if (row0 + r >= m4) continue;
    const float* src = partial + (size_t)(row0 + r) * bpad + beta;
    float v = 0.f;
    for (int s = 0; s < S2; ++s) v += __ldcg(src + (size_t)s * m4 * bpad);
    tile[beta][r] = v;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < b * 64; e += 256) {
    const int beta = e / 64, r = e % 64;
    if (row0 + r >= m) continue;
    const size_t o = (size_t)beta * m + row0 + r;
    if (yf) yf[o] = tile[beta][r];
    else y[o] = __float2half_rn(tile[beta][r]);
  }
}

// ---------------------------------------------------------------------------
// Cross-slice reduction: Y[beta][r] = sum_{s=0}^{S-1} partial[s][beta][r] in
// slice order (deterministic, R11), then fp16 round-to-nearest-even (or fp32).
// One thread per (beta, row quad); launched with PDL after the LUT kernel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lut_reduce_kernel(const float* __restrict__ partial, int S, int b, int m,
                                                         int m4, __half* __restrict__ y, float* __restrict__ yf) {
  pdl_launch_dependents();  // the next product may start streaming its weights
  pdl_wait();               // partials are complete and visible
  const int RQ = m4 / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= b * RQ) return;
  const int beta = idx / RQ, rq = idx % RQ;
  const float4* src = reinterpret_cast<const float4*>(partial + (size_t)beta * m4) + rq;
  const size_t stride = (size_t)b * RQ;  // float4 units between slices
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int s0 = 0; s0 < S; s0 += 8) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (s0 + k < S) ? __ldcg(src + (size_t)(s0 + k) * stride) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (s0 + k < S) {
        acc.x += v[k].x;
        acc.y += v[k].y;
        acc.z += v[k].z;
        acc.w += v[k].w;
      }
  }
  const float r[4] = {acc.x, acc.y, acc.z, acc.w};
  const int row0 = 4 * rq;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (row0 + k < m) {
      const size_t o = (size_t)beta * m + row0 + k;
      if (yf) yf[o] = r[k];
      else y[o] = __float2half_rn(r[k]);
    }
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

// the dynamic shared-memory opt-in, set once per (kernel, device) instead of on every launch
static cudaError_t ensure_smem_attr(const void* kernel) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& d : done)
    if (d.first == kernel && d.second == dev) return cudaSuccess;
  const cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (err == cudaSuccess) done.emplace_back(kernel, dev);
  return err;
}

static cudaLaunchAttribute g_pdl_attr = [] {
  cudaLaunchAttribute a;
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  return a;
}();

std::atomic<unsigned long long> g_launches{0};  // product kernels launched by this process (lutgemm_launch_count)

template <typename K>
static cudaError_t launch(K kernel, int grid, const KParams& p, cudaStream_t st, int threads = kThreads) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t err = ensure_smem_attr(reinterpret_cast<const void*>(kernel));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cfg.attrs = &g_pdl_attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

static cudaError_t launch_reduce(const KParams& p, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static bool attr_set = false;
  if (!attr_set) {  // keep the max-shared-memory carveout: no L1/smem reconfiguration between the two kernels
    cudaFuncSetAttribute(lut_reduce_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr_set = true;
  }
  const int threads = 256;
  const int total = p.b * p.sh.RQ;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((total + threads - 1) / threads);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cfg.attrs = &g_pdl_attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lut_reduce_kernel, (const float*)p.partial, p.sh.S, p.b, p.sh.m, p.sh.m4, p.y,
                            p.yf);
}

template <int QT, int ZM>
static cudaError_t launch_gemv_t(const KParams& p, int grid, cudaStream_t st) {
  // quads in flight per warp while one is computed (ring of PD + 1 buffers)
  constexpr int PD = QT <= 1 ? 6 : (QT <= 2 ? 4 : (QT <= 4 ? 2 : 1));
  return launch(lut_gemv_kernel<QT, ZM, PD>, grid, p, st);
}

template <int QT, int ZM>
static cudaError_t launch_gemvv_t(const KParams& p, int grid, cudaStream_t st) {
  constexpr int PD = QT <= 2 ? 3 : (QT <= 4 ? 2 : 1);
  if (p.b == 2) return launch(lut_gemvv_kernel<2, QT, ZM, PD>, grid, p, st);
  return launch(lut_gemvv_kernel<4, QT, ZM, PD>, grid, p, st);
}

// batched: V-wide slots (V = 2 only for b = 2); p.qpw = row quads per work item
// (256 or 128).  V = 2 runs 16 warps (128 registers: 4 rows x 2 batch x 16
// quads of accumulators), V = 4 and q > 4 run 8 warps (255 registers).
template <int V, int QT, int ZM>
static cudaError_t launch_batched_v(const KParams& p, int grid, cudaStream_t st) {
  if constexpr (QT <= 4 && V == 2) {
    if (p.qpw == 128) return launch(lut_gemm_batched_kernel<V, QT, ZM, 1, 8, 512>, grid, p, st, 512);
    return launch(lut_gemm_batched_kernel<V, QT, ZM, 1, 16, 512>, grid, p, st, 512);
  } else if constexpr (QT <= 4) {
    if (p.qpw == 128) return launch(lut_gemm_batched_kernel<V, QT, ZM, 1, 16, 256>, grid, p, st, 256);
    return launch(lut_gemm_batched_kernel<V, QT, ZM, 1, 32, 256>, grid, p, st, 256);
  } else {
    return launch(lut_gemm_batched_kernel<V, QT, ZM, 1, 16, 256>, grid, p, st, 256);
  }
}

template <int QT, int ZM>
static cudaError_t launch_batched_t(const KParams& p, int grid, cudaStream_t st) {
  if (p.s2 > 0) return launch_gemvv_t<QT, ZM>(p, grid, st);
  return p.b == 2 ? launch_batched_v<2, QT, ZM>(p, grid, st) : launch_batched_v<4, QT, ZM>(p, grid, st);
}

static cudaError_t launch_reduce_batched(const KParams& p, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.sh.m4 + 63) / 64);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = &g_pdl_attr;
  cfg.numAttrs = 1;
  const int S2 = (p.sh.S + p.spi - 1) / p.spi;
  return cudaLaunchKernelEx(&cfg, lut_reduce_batched_kernel, (const float*)p.partial, S2, p.b, 1 << p.bl, p.sh.m,
                            p.sh.m4, p.y, p.yf);
}

// Work split of the batched kernel: items = (range of spi slices, row block of
// rbq = 256 or 128 quads); pick (rbq, spi) minimising waves * spi * (per-sub-
// slice lookup time + LUT rebuild time), ties to fewer partials (larger spi).
static void plan_batched(const Shape& sh, int sms, KParams& p) {
  double best = 1e30;
  const int rbqs[2] = {256, 128};
  static int force = -1;
  if (force < 0) {
    const char* env = getenv("LUTGEMM_BRBQ");  // tuning knob: force 256 or 128
    force = env ? atoi(env) : 0;
  }
  for (int qi = 0; qi < 2; ++qi) {
    const int rbq = rbqs[qi];
    if ((sh.q > 4 && rbq != 128) || (force && rbq != force)) continue;
    const long long nrb = (sh.RQ + rbq - 1) / rbq;
    for (int spi = 1; spi <= sh.S; ++spi) {
      const long long items = (long long)((sh.S + spi - 1) / spi) * nrb;
      const long long waves = (items + sms - 1) / sms;
      const double cost = (double)waves * spi * (rbq * 16.0 * sh.q + 1200.0);
      if (cost < best * 0.999 || (cost <= best * 1.001 && spi > p.spi)) {
        best = std::min(best, cost);
        p.qpw = rbq;
        p.spi = spi;
        p.items = items;
      }
    }
  }
}

template <int ZM>
static cudaError_t dispatch_q(const KParams& p, int grid, cudaStream_t st, bool batched) {
  switch (p.sh.q) {
    case 1: return batched ? launch_batched_t<1, ZM>(p, grid, st) : launch_gemv_t<1, ZM>(p, grid, st);
    case 2: return batched ? launch_batched_t<2, ZM>(p, grid, st) : launch_gemv_t<2, ZM>(p, grid, st);
    case 3: return batched ? launch_batched_t<3, ZM>(p, grid, st) : launch_gemv_t<3, ZM>(p, grid, st);
    case 4: return batched ? launch_batched_t<4, ZM>(p, grid, st) : launch_gemv_t<4, ZM>(p, grid, st);
    default: return batched ? launch_batched_t<8, ZM>(p, grid, st) : launch_gemv_t<8, ZM>(p, grid, st);
  }
}

static size_t counters_bytes(const Shape&) { return 2u * kFusedMaxJ * 4u; }

int batch_pad(int b) {
  int bp = 1;
  while (bp < b) bp <<= 1;
  return b == 1 ? 1 : (b == 2 ? 2 : std::max(bp, 4));
}

size_t workspace_bytes(const Shape& sh, int b) {
  // b <= 4: sub-slice partials of the GEMV-structured kernel ([V S][b][m4], V = 2 or 4)
  const size_t slices = b == 2 ? 2 * (size_t)sh.S : (b <= 4 && b > 1 ? 4 * (size_t)sh.S : (size_t)sh.S);
  return counters_bytes(sh) + (slices * (size_t)batch_pad(b) * (size_t)sh.m4 * 4u + 255) / 256 * 256;
}

static unsigned long long* g_trace = nullptr;
static bool g_trace_on = false;
constexpr int kTraceMaxCtas = 1024;

unsigned long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

void trace_enable(int on) {
  g_trace_on = on != 0;
  if (g_trace_on && !g_trace) cudaMalloc(&g_trace, sizeof(unsigned long long) * kTraceSlots * kTraceMaxCtas);
  if (g_trace_on && g_trace) cudaMemset(g_trace, 0, sizeof(unsigned long long) * kTraceSlots * kTraceMaxCtas);
}

size_t trace_read(unsigned long long* host, size_t n) {
  if (!g_trace || !host) return 0;
  const size_t cap = (size_t)kTraceSlots * kTraceMaxCtas;
  if (n > cap) n = cap;
  cudaMemcpy(host, g_trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return n;
}

// fused mode of the GEMV-structured kernels: S slices x J CTAs with J = #SMs / S,
// idling at most 8 % of the SMs, and at least J row units per slice
static bool fusable(int S, int units, int sms) {
  const int J = S <= sms ? sms / S : 0;
  return J >= 1 && J <= kFusedMaxJ && S <= kFusedMaxJ && S * J * 100 >= sms * 92 && units >= J;
}

cudaError_t run_product(const Shape& sh, const void* data, const uint16_t* x, int b, uint16_t* y, float* yf,
                        void* ws, cudaStream_t st) {
  KParams p;
  p.data = static_cast<const uint8_t*>(data);
  p.x = reinterpret_cast<const __half*>(x);
  p.y = reinterpret_cast<__half*>(y);
  p.yf = yf;
  p.counters = static_cast<unsigned*>(ws);
  p.partial = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + counters_bytes(sh));
  p.sh = sh;
  p.b = b;
  int bl = 0;
  while ((1 << bl) < batch_pad(b)) ++bl;
  p.bl = bl;
  p.nv = b == 2 ? 1 : (1 << bl) / 4;
  p.spi = 1;
  p.qpw = 256;
  {
    int gs = 0;  // layout lane -> group shift (lanes are 32 columns); g > 1024: one group per slice
    while (gs < 5 && (32 << gs) < sh.g) ++gs;
    p.gsh = sh.g <= kSliceCols ? gs : 31;
  }
  {
    static unsigned seq = 0;  // consecutive launches alternate between two halves of the trace buffer
    p.trace = g_trace_on ? g_trace + (size_t)(seq++ & 1u) * (kTraceMaxCtas / 2) * kTraceSlots : nullptr;
  }
  const bool batched = b > 1;
  p.s2 = 0;
  if (!batched) {
    p.items = (long long)sh.S * sh.RQ;
  } else if (b <= 4 && !(getenv("LUTGEMM_SMALLB_BATCHED") && atoi(getenv("LUTGEMM_SMALLB_BATCHED")))) {
    // b <= 4: GEMV-structured kernel over sub-slices of 1024 / V columns, V = 2 (b = 2)
    // or 4 (b = 3, 4); LUTGEMM_SMALLB_BATCHED=1 selects the vector-slot batched kernel
    const int V = b == 2 ? 2 : 4;
    p.s2 = (sh.n + 1024 / V - 1) / (1024 / V);
    p.items = (long long)p.s2 * ((sh.RQ + V - 1) / V);
  } else {
    p.spi = 0;
    plan_batched(sh, num_sms(), p);
  }
  int grid = (int)std::min<long long>((long long)num_sms(), p.items);
  // fused mode (b = 1): whole slices per CTA group, S*J CTAs with J per slice,
  // when that idles at most 8 % of the SMs; the reduction then runs in-kernel
  // with R reducers per row-quad group (~16 KB of partials each; the others
  // exit early).  LUTGEMM_GEMV_REDUCERS overrides R (tests, tuning).
  p.fused_J = 0;
  p.reducers = 0;
  if (p.s2 > 0) {  // b <= 4 kernel: the GEMV's fused mode over sub-slices
    const int sms = num_sms();
    const int V = b == 2 ? 2 : 4;
    const int NG = (sh.RQ + V - 1) / V;
    const int J = p.s2 <= sms ? sms / p.s2 : 0;
    if (fusable(p.s2, NG, sms)) {
      p.fused_J = J;
      grid = p.s2 * J;
      const long long red_bytes = (long long)p.s2 * b * 4 * (4 * V) * ((NG + J - 1) / J);
      p.reducers = (int)std::min<long long>(p.s2, (red_bytes + 16383) / 16384);
    }
  }
  if (!batched) {
    const int sms = num_sms();
    const int J = sh.S <= sms ? sms / sh.S : 0;
    if (fusable(sh.S, sh.RQ, sms)) {
      p.fused_J = J;
      grid = sh.S * J;
      const long long red_bytes = (long long)sh.S * 16 * ((sh.RQ + J - 1) / J);
      p.reducers = (int)std::min<long long>(sh.S, (red_bytes + 16383) / 16384);
      const char* env = getenv("LUTGEMM_GEMV_REDUCERS");
      if (env && atoi(env) > 0) p.reducers = std::min(atoi(env), sh.S);
    }
  }
  cudaError_t e = sh.compact ? dispatch_q<2>(p, grid, st, batched)
                             : (sh.has_z ? dispatch_q<1>(p, grid, st, batched) : dispatch_q<0>(p, grid, st, batched));
  if (e != cudaSuccess) return e;
  if (p.fused_J > 0) return cudaSuccess;  // reduced in-kernel
  if (p.s2 > 0) {  // sub-slice partials [SV][b][m4]: the GEMV reduction kernel with S = SV
    KParams r = p;
    r.sh.S = p.s2;
    return launch_reduce(r, st);
  }
  return batched ? launch_reduce_batched(p, st) : launch_reduce(p, st);
}

}  // namespace lg
