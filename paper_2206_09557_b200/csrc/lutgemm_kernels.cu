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
//  * the weight is one slice-major record stream (layout.cuh); one thread
//    keeps a bulk L2 prefetch (TMA engine, UBLKPF) several row-quad steps
//    ahead of the warps, whose 128-bit loads (L1::no_allocate) then hit L2;
//    a PD-deep register ring overlaps those loads with the lookups;
//  * the activation slice is staged into shared memory by the bulk-copy
//    (TMA) engine, double-buffered one segment ahead;
//  * lookups summed and scaled with packed f32x2 adds/FMAs (FADD2/FFMA2),
//    two rows per instruction;
//  * per-row partials reduced across lanes by a 6-shuffle transpose-reduce and
//    written to an fp32 split-K workspace; a small second kernel, chained by
//    programmatic dependent launch (PDL), sums the slices in fixed order
//    (deterministic) and rounds y to fp16.  The LUT kernel streams its first
//    weights before griddepcontrol.wait, so back-to-back products overlap.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "layout.cuh"
#include "lutgemm_internal.h"
#include "ptx.cuh"

namespace lg {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kQPW = 9;                // batched: row quads per warp per work item (multiple of the ring size)
constexpr int kMiscBytes = 8192;       // x double buffer (2 x 2 KB) + mbarriers + flags
constexpr int kSmemBytes = 3 * 65536;  // LUT (128 KB) on a 64 KB boundary + misc, for any base
constexpr int kPfSteps = 8;            // GEMV: L2 prefetch distance in 16-quad steps
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
// MODE != 0 are measurement variants (tools/kernel_probe): 1 = no LDS.
template <int J, int MODE = 0>
__device__ __forceinline__ float lut1(uint32_t w, uint32_t lc) {
  constexpr uint32_t kSel = ((J & 1) ? 0x7605u : 0x7604u) | ((uint32_t)J << 4);
  if (MODE == 1) return __uint_as_float(prmt<kSel>(w, lc) & 0x3fffffffu);
  return lds_f32<(J >> 1) * 65536>(prmt<kSel>(w, lc));
}

// sum over the 4 keys of word wa (row a) and of word wb (row b), as the pair (a, b)
template <int MODE = 0>
__device__ __forceinline__ f32x2 lut4x2(uint32_t wa, uint32_t wb, uint32_t lc) {
  const f32x2 p0 = pack2(lut1<0, MODE>(wa, lc), lut1<0, MODE>(wb, lc));
  const f32x2 p1 = pack2(lut1<1, MODE>(wa, lc), lut1<1, MODE>(wb, lc));
  const f32x2 p2 = pack2(lut1<2, MODE>(wa, lc), lut1<2, MODE>(wb, lc));
  const f32x2 p3 = pack2(lut1<3, MODE>(wa, lc), lut1<3, MODE>(wb, lc));
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

// L2 prefetch of row quads [a, b) of slice s (all regions), issued by one thread
__device__ __forceinline__ void prefetch_quads(const Shape& sh, const uint8_t* data, int s, int Ls, int a, int b) {
  if (b <= a) return;
  const uint32_t kb = keys_bytes(sh, Ls), ab = alpha_bytes(sh, Ls), zb = z_bytes(sh, Ls);
  // region starts are 256-aligned; per-quad sizes are multiples of 8, so round the ranges to 16 bytes
  auto pf = [](const uint8_t* base, size_t lo, size_t hi) {
    lo &= ~(size_t)15;
    hi = (hi + 15) & ~(size_t)15;
    if (hi > lo) bulk_prefetch_l2(base + lo, (uint32_t)(hi - lo));
  };
  pf(data + keys_base(sh, s, Ls), (size_t)a * kb, (size_t)b * kb);
  pf(data + alpha_base(sh, s, Ls), (size_t)a * ab, (size_t)b * ab);
  if (zb) pf(data + z_base(sh, s, Ls), (size_t)a * zb, (size_t)b * zb);
}

template <int QT, bool HAS_Z, int MODE = 0>
__device__ __forceinline__ void ring_load(Ring<QT>& r, bool ok, const LaneAddr& la, int rq, int q) {
  if (ok) {
    const uint8_t* kp = la.kp + (size_t)rq * la.KB;
    const uint8_t* ap = la.ap + (size_t)rq * la.AB;
#pragma unroll
    for (int i = 0; i < QT; ++i) {
      if (QT <= 4 || i < q) {
        r.k[i] = ldg_stream_u4(kp + i * la.kstride);
        if (MODE != 4) r.a[i] = ldg_nc_u2(ap + 8 * i);
        else r.a[i] = make_uint2(0, 0);
      }
    }
    if (HAS_Z) r.z = ldg_nc_u2(la.zp + (size_t)rq * la.ZB);
  } else {
#pragma unroll
    for (int i = 0; i < QT; ++i) {
      r.k[i] = make_uint4(0, 0, 0, 0);
      r.a[i] = make_uint2(0, 0);
    }
    r.z = make_uint2(0, 0);
  }
}

// (acc01, acc23) (+)= sum_i alpha_i[r] * (LUT partial of row r, plane i) (+ z[r] * xsum)
template <int QT, bool HAS_Z, int MODE = 0>
__device__ __forceinline__ void ring_compute(const Ring<QT>& r, uint32_t lc, float xsum, f32x2& acc01, f32x2& acc23,
                                             int q, bool accumulate) {
  if (MODE == 3 || MODE == 4) {  // measurement variants: consume the loaded words with minimal work
    uint32_t v = 0;
#pragma unroll
    for (int i = 0; i < QT; ++i) v ^= r.k[i].x ^ r.k[i].y ^ r.k[i].z ^ r.k[i].w ^ r.a[i].x ^ r.a[i].y;
    acc01 = pack2(__uint_as_float(v & 0x3fffffffu), 0.f);
    acc23 = pack2(0.f, 0.f);
    return;
  }
#pragma unroll
  for (int i = 0; i < QT; ++i) {
    if (QT <= 4 || i < q) {
      const f32x2 a01 = h2_to_f32x2(r.a[i].x), a23 = h2_to_f32x2(r.a[i].y);
      const f32x2 s01 = lut4x2<MODE>(r.k[i].x, r.k[i].y, lc);
      const f32x2 s23 = lut4x2<MODE>(r.k[i].z, r.k[i].w, lc);
      if (i == 0 && !accumulate) {
        acc01 = mul2(a01, s01);
        acc23 = mul2(a23, s23);
      } else {
        acc01 = fma2(a01, s01, acc01);
        acc23 = fma2(a23, s23, acc23);
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
// Work distribution: the S*RQ (slice, row-quad) items are split into equal
// contiguous ranges, one per CTA (a range spans at most a few slices, so a CTA
// builds few LUTs).  Inside a range the 16 warps take row quads round-robin.
// ---------------------------------------------------------------------------
template <int QT, bool HAS_Z, int PD, int MODE = 0>
__global__ void __launch_bounds__(kThreads, 1) lut_gemv_kernel(const KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);  // warp-uniform for the compiler
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  // work: a contiguous range of the S*RQ (slice, row-quad) items; in the fused
  // mode CTA c owns slice c / J, row-quad group c % J (one segment)
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

  const SmemMap sm = map_smem(smem);
  __half* xbuf0 = reinterpret_cast<__half*>(sm.misc_p);
  __half* xbuf1 = reinterpret_cast<__half*>(sm.misc_p + 2048);
  const uint32_t bar0 = sm.misc + 4096, bar1 = sm.misc + 4104;
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)(4 * lane + 128) << 8) | (uint32_t)(4 * lane);
  const int pf_steps = p.pf_steps;

  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar1, 1);
    fence_mbar_init();
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
    const LaneAddr la = lane_addr(sh, p.data, s, Ls, lane_ok ? lane : 0);

    // 1. the x slice of the first segment (after the PDL wait: x belongs to the
    //    preceding kernel until it completes) is requested before anything
    //    else, so it is not queued behind the weight stream; then an L2
    //    prefetch of the first weight steps and the register ring
    if (e == 0) {
      // weights of the steps after the register prologue into L2 while the
      // preceding kernel drains (a plain prefetch: legal before the PDL wait)
      if (tid == 0 && p.pf_init > PD)
        prefetch_quads(sh, p.data, s, Ls, min(rq_b, rq_a + PD * kWarps), min(rq_b, rq_a + p.pf_init * kWarps));
      pdl_wait();
      if (trace) trace[5] = globaltimer_ns();
      if (warp == 0) stage_x(xbuf0, bar0, p.x, sh.n, s * kSliceCols, Ls, 32, 1, 1, lane);
    }
    if (tid == 0 && pf_steps > 0) prefetch_quads(sh, p.data, s, Ls, rq_a, min(rq_b, rq_a + pf_steps * kWarps));
    // this warp's row quads in the segment: rq_a + warp + 16 t, t < nt
    const int nt = rq_a + warp < rq_b ? (rq_b - (rq_a + warp) + kWarps - 1) / kWarps : 0;
    // a ring of NB = PD + 1 single-quad buffers: the load for quad t + PD is
    // issued BEFORE quad t is computed (the lookups and the reduction's
    // shuffles would otherwise delay it), so PD quads are always in flight
    constexpr int NB = PD + 1;
    Ring<QT> buf[NB];
    auto load_quad = [&](Ring<QT>& b, int t) {
      ring_load<QT, HAS_Z, MODE>(b, lane_ok && t < nt, la, rq_a + warp + kWarps * t, q);
    };
#pragma unroll
    for (int d = 0; d < PD; ++d) load_quad(buf[d], d);
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
    float* part = p.partial + (size_t)s * sh.m4;
    // 4. main loop
    for (int t0 = 0; t0 < nt; t0 += NB) {
      if (tid == 0 && pf_steps > 0) {  // optional L2 prefetch pf_steps steps ahead of warp 0
        const int lo = rq_a + kWarps * (t0 + pf_steps);
        prefetch_quads(sh, p.data, s, Ls, lo, min(rq_b, lo + NB * kWarps));
      }
#pragma unroll
      for (int d = 0; d < NB; ++d) {
        const int t = t0 + d;
        if (t < nt) {
          load_quad(buf[(d + PD) % NB], t + PD);
          const int rq = rq_a + warp + kWarps * t;
          f32x2 acc01, acc23;
          ring_compute<QT, HAS_Z, MODE>(buf[d], lc, xsum, acc01, acc23, q, false);
          const float v = reduce4(acc01, acc23, lane);
          if ((lane & 7) == 0) part[4 * rq + (lane >> 3)] = v;
        }
      }
    }
    if (trace && e == 0) trace[3] = globaltimer_ns();  // warp 0's loop end
    if (J > 0) {  // fused mode: each warp publishes its partials with one release increment
      __syncwarp();
      if (lane == 0) red_release_add_u32(p.counters + blockIdx.x % J, 1u);
    }
    __syncthreads();  // the LUT and x buffer are reused by the next segment
    if (trace) trace[e == 0 ? 4 : 6] = globaltimer_ns();  // all warps done
    it = itn;
    ++e;
  }
  if (trace) trace[7] |= (unsigned long long)e << 32;  // segments processed
  if (J > 0) {
    // Fused cross-slice reduction: the S CTAs that share row-quad group fj
    // (one per slice) meet at a counter -- all CTAs of the grid are resident
    // (grid <= #SMs, one CTA per SM) -- then each sums its 1/S share of the
    // group's rows over the S slices in slice order (deterministic, R11).
    const int fs = blockIdx.x / J, fj = blockIdx.x % J;
    unsigned* arrive = p.counters + fj;
    unsigned* depart = p.counters + kFusedMaxJ + fj;
    if (e == 0) {  // an empty range never reached the wait and the warp increments above
      pdl_wait();
      if (lane == 0) red_release_add_u32(arrive, 1u);
    }
    if (tid == 0) {  // all 16 warps of all S CTAs of the group have published their partials
      while (ld_acquire_u32(arrive) < (unsigned)(sh.S * kWarps)) __nanosleep(32);
    }
    __syncthreads();
    if (trace) trace[5] = globaltimer_ns();  // (re-used) the group is complete
    const int g0 = (int)((long long)sh.RQ * fj / J), g1 = (int)((long long)sh.RQ * (fj + 1) / J);
    const int r0 = 4 * (g0 + (int)((long long)(g1 - g0) * fs / sh.S));
    const int r1 = min(sh.m, 4 * (g0 + (int)((long long)(g1 - g0) * (fs + 1) / sh.S)));
    for (int r = r0 + tid; r < r1; r += kThreads) {
      float v = 0.f;
      const float* pp = p.partial + r;
      for (int ss0 = 0; ss0 < sh.S; ss0 += 16) {  // up to 16 slices per L2 round trip
        float t[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) t[k] = (ss0 + k < sh.S) ? __ldcg(pp + (size_t)(ss0 + k) * sh.m4) : 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (ss0 + k < sh.S) v += t[k];
      }
      if (p.yf) p.yf[r] = v;
      else p.y[r] = __float2half_rn(v);
    }
    __syncthreads();
    if (tid == 0 && atomicAdd(depart, 1u) == (unsigned)sh.S - 1) {  // the last one resets the pair
      *arrive = 0u;
      *depart = 0u;
    }
    if (trace) trace[6] = globaltimer_ns();  // reduction share done
  }
  pdl_launch_dependents();  // the next kernel may now be scheduled
}

// ---------------------------------------------------------------------------
// Batched LUT-GEMM, 2 <= b <= 32.  B = 2^bl >= b table banks
// share each key: lane l = (pp = l >> bl, beta = l & (B-1)); a CTA's 128
// tables hold P = 32/B layout lanes x 4 chunks x B batch rows, so a native
// slice is processed as B sub-slices with register accumulators across them.
// ---------------------------------------------------------------------------
template <int QT, bool HAS_Z, int PD, int QPW>
__global__ void __launch_bounds__(kThreads, 1) lut_gemm_batched_kernel(const KParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  const int bl = p.bl, B = 1 << bl, P = 32 >> bl, b = p.b;
  const int beta = lane & (B - 1), pp = lane >> bl;
  constexpr int NB = PD + 1;  // ring buffers; loads for quad t+PD issued before quad t's lookups
  static_assert(QPW % NB == 0, "the ring restarts at buffer 0 every sub-slice");
  const int rbq = kWarps * QPW;  // row quads per work item
  const int NRB = (sh.RQ + rbq - 1) / rbq;
  const long long it0 = p.items * blockIdx.x / gridDim.x;
  const long long it1 = p.items * (blockIdx.x + 1) / gridDim.x;
  if (it0 >= it1) return;

  const SmemMap sm = map_smem(smem);
  // two x tiles [B][32P] fp16 (2 KB each), filled by cp.async one sub-slice ahead
  const __half* xtile0 = reinterpret_cast<const __half*>(sm.misc_p);
  const __half* xtile1 = reinterpret_cast<const __half*>(sm.misc_p + 2048);
  const uint32_t xt0 = sm.misc, xt1 = sm.misc + 2048;
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)(4 * lane + 128) << 8) | (uint32_t)(4 * lane);

  // x tile of sub-slice (itx, k) -- x[beta][col0 .. col0 + 32P) for every
  // table bank beta, zero for beta >= b and lanes past the slice end -- one
  // 16-byte cp.async per thread for the first 128 threads (x is L2-resident)
  auto load_x = [&](uint32_t dst, long long itx, int k) {
    if (tid < 128) {
      const int s = (int)(itx / NRB);
      const int Ls = slice_lanes(sh.n, s);
      const int bt = tid / (4 * P), c = tid % (4 * P);  // row of the tile, 16-byte chunk in the row
      const bool ok = bt < b && k * P + c / 4 < Ls;
      const __half* src = ok ? p.x + (size_t)bt * sh.n + s * kSliceCols + 32 * k * P + 8 * c : p.x;
      cp_async_16(dst + 16u * tid, src, ok ? 16u : 0u);
    }
  };
  // the (item, sub-slice) after (itx, k)
  auto advance = [&](long long& itx, int& k) {
    const int Ls = slice_lanes(sh.n, (int)(itx / NRB));
    if (++k >= (Ls + P - 1) / P) {
      k = 0;
      ++itx;
    }
  };
  Ring<QT> ring[NB];
  // first PD quads of sub-slice (itx, k) for this warp into ring[0..PD)
  auto prologue = [&](long long itx, int k) {
    const int s = (int)(itx / NRB), rb = (int)(itx % NRB);
    const int Ls = slice_lanes(sh.n, s);
    const int lay = k * P + pp;
    const bool ok = lay < Ls;
    const LaneAddr la = lane_addr(sh, p.data, s, Ls, ok ? lay : 0);
    const int rq_w = rb * rbq + warp * QPW;
#pragma unroll
    for (int d = 0; d < PD; ++d) ring_load<QT, HAS_Z>(ring[d], ok && rq_w + d < sh.RQ, la, rq_w + d, q);
  };

  prologue(it0, 0);  // weights only: legal before the PDL wait
  pdl_wait();        // x and the workspace belong to the preceding kernel until it completes
  load_x(xt0, it0, 0);
  cp_async_wait_all();
  __syncthreads();
  int e = 0;  // sub-slices processed: x tile e & 1

  for (long long it = it0; it < it1; ++it) {
    const int s = (int)(it / NRB);
    const int rb = (int)(it % NRB);
    const int Ls = slice_lanes(sh.n, s);
    const int nsub = (Ls + P - 1) / P;
    const int rq_w = rb * rbq + warp * QPW;  // this warp's first quad
    f32x2 acc01[QPW], acc23[QPW];

    for (int k = 0; k < nsub; ++k, ++e) {
      unsigned long long* tr = (p.trace && tid == 0 && it == it0 && k >= 2 && k < 4)
                                   ? p.trace + (size_t)blockIdx.x * kTraceSlots + 4 * (k - 2) : nullptr;
      if (tr) tr[0] = globaltimer_ns();
      const int lay = k * P + pp;
      const bool lane_ok = lay < Ls;
      const LaneAddr la = lane_addr(sh, p.data, s, Ls, lane_ok ? lay : 0);
      if (tr) tr[1] = globaltimer_ns();
      {
        const int l = lane, j = warp & 3, h = warp >> 2;
        const int bt = l & (B - 1), pl = l >> bl;
        build_table_part(sm.lut + table_offset(l, j), ((e & 1) ? xtile1 : xtile0) + (size_t)bt * 32 * P + (4 * pl + j) * 8,
                         h);
      }
      __syncthreads();
      if (tr) tr[2] = globaltimer_ns();
      long long itn = it;
      int kn = k;
      advance(itn, kn);
      if (itn < it1) load_x((e & 1) ? xt0 : xt1, itn, kn);  // lands during the lookups
      const float xsum = (HAS_Z && lane_ok) ? lane_xsum(sm.lut, lane) : 0.f;
#pragma unroll
      for (int t = 0; t < QPW; ++t) {
        if (t + PD < QPW)
          ring_load<QT, HAS_Z>(ring[(t + PD) % NB], lane_ok && rq_w + t + PD < sh.RQ, la, rq_w + t + PD, q);
        ring_compute<QT, HAS_Z>(ring[t % NB], lc, xsum, acc01[t], acc23[t], q, k > 0);
      }
      if (itn < it1) prologue(itn, kn);  // next sub-slice's first quads fly during the barrier and rebuild
      if (tr) tr[3] = globaltimer_ns();
      cp_async_wait_all();
      __syncthreads();  // every warp is done with the LUT; the next x tile is visible
    }
    // reduce over the P layout lanes that share a batch row (lane bits >= bl)
#pragma unroll
    for (int t = 0; t < QPW; ++t) {
      float2 v01 = unpack2(acc01[t]), v23 = unpack2(acc23[t]);
      for (int off = 16; off >= B; off >>= 1) {
        v01.x += __shfl_xor_sync(kFull, v01.x, off);
        v01.y += __shfl_xor_sync(kFull, v01.y, off);
        v23.x += __shfl_xor_sync(kFull, v23.x, off);
        v23.y += __shfl_xor_sync(kFull, v23.y, off);
      }
      const int rq = rq_w + t;
      if (pp == 0 && beta < b && rq < sh.RQ) {
        float* dst = p.partial + ((size_t)s * b + beta) * sh.m4 + 4 * rq;
        *reinterpret_cast<float4*>(dst) = make_float4(v01.x, v01.y, v23.x, v23.y);
      }
    }
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// Cross-slice reduction: Y[beta][r] = sum_{s=0}^{S-1} partial[s][beta][r] in
// slice order (deterministic, R11), then fp16 round-to-nearest-even (or fp32).
// One thread per (beta, row quad); launched with PDL after the LUT kernel.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lut_reduce_kernel(const float* __restrict__ partial, int S, int b, int m,
                                                         int m4, __half* __restrict__ y, float* __restrict__ yf,
                                                         unsigned* __restrict__ counters) {
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

static cudaLaunchAttribute g_pdl_attr = [] {
  cudaLaunchAttribute a;
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  return a;
}();

template <typename K>
static cudaError_t launch(K kernel, int grid, const KParams& p, cudaStream_t st) {
  cudaError_t err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cfg.attrs = &g_pdl_attr;
  cfg.numAttrs = p.xmode == 3 ? 0 : 1;  // experiment 3: no PDL
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

static cudaError_t launch_reduce(const KParams& p, cudaStream_t st) {
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
  cfg.numAttrs = p.xmode == 3 ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, lut_reduce_kernel, (const float*)p.partial, p.sh.S, p.b, p.sh.m, p.sh.m4, p.y,
                            p.yf, p.counters);
}

template <int QT, bool HAS_Z>
static cudaError_t launch_gemv_t(const KParams& p, int grid, cudaStream_t st) {
  // quads in flight per warp while one is computed (ring of PD + 1 buffers)
  constexpr int PD = QT <= 1 ? 6 : (QT <= 2 ? 4 : (QT <= 4 ? 2 : 1));
  if constexpr (QT == 3 && !HAS_Z) {
    if (p.xmode >= 10) {  // measurement variants (LUTGEMM_XMODE)
    switch (p.xmode) {
      case 10: return launch(lut_gemv_kernel<QT, HAS_Z, 1, 0>, grid, p, st);
      case 11: return launch(lut_gemv_kernel<QT, HAS_Z, 2, 1>, grid, p, st);
      case 13: return launch(lut_gemv_kernel<QT, HAS_Z, 2, 3>, grid, p, st);
      case 16: return launch(lut_gemv_kernel<QT, HAS_Z, 2, 4>, grid, p, st);
      case 14: return launch(lut_gemv_kernel<QT, HAS_Z, 3, 0>, grid, p, st);
      case 18: return launch(lut_gemv_kernel<QT, HAS_Z, 4, 0>, grid, p, st);
      default: break;
    }
    }
  }
  return launch(lut_gemv_kernel<QT, HAS_Z, PD>, grid, p, st);
}

static int batched_qpw(const KParams& p) { return p.xmode == 6 ? 6 : (p.xmode == 7 ? 8 : kQPW); }

template <int QT, bool HAS_Z>
static cudaError_t launch_batched_t(const KParams& p, int grid, cudaStream_t st) {
  constexpr int PD = QT <= 4 ? 2 : 0;  // QPW % (PD + 1) == 0
  if constexpr (QT <= 4) {
    if (p.xmode == 6) return launch(lut_gemm_batched_kernel<QT, HAS_Z, PD, 6>, grid, p, st);
    if (p.xmode == 7) return launch(lut_gemm_batched_kernel<QT, HAS_Z, 1, 8>, grid, p, st);
  }
  return launch(lut_gemm_batched_kernel<QT, HAS_Z, PD, kQPW>, grid, p, st);
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

static size_t counters_bytes(const Shape&) { return 2u * kFusedMaxJ * 4u; }

size_t workspace_bytes(const Shape& sh, int b) {
  return counters_bytes(sh) + ((size_t)sh.S * (size_t)b * (size_t)sh.m4 * 4u + 255) / 256 * 256;
}

static int g_pf_steps = -1;
static unsigned long long* g_trace = nullptr;
static bool g_trace_on = false;
constexpr int kTraceMaxCtas = 1024;

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

cudaError_t run_product(const Shape& sh, const void* data, const uint16_t* x, int b, uint16_t* y, float* yf,
                        void* ws, cudaStream_t st) {
  if (g_pf_steps < 0) {
    const char* env = getenv("LUTGEMM_PF_STEPS");  // tuning knob (default kPfSteps)
    g_pf_steps = env ? atoi(env) : 0;
  }
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
  while ((1 << bl) < b) ++bl;
  p.bl = bl;
  p.pf_steps = g_pf_steps;
  {
    static int pf_init = -1;
    if (pf_init < 0) {
      const char* env = getenv("LUTGEMM_PF_INIT");  // tuning knob
      pf_init = env ? atoi(env) : 0;
    }
    p.pf_init = pf_init;
  }
  {
    const char* env = getenv("LUTGEMM_XMODE");  // experiment knob
    p.xmode = env ? atoi(env) : 0;
  }
  {
    static unsigned seq = 0;  // consecutive launches alternate between two halves of the trace buffer
    p.trace = g_trace_on ? g_trace + (size_t)(seq++ & 1u) * (kTraceMaxCtas / 2) * kTraceSlots : nullptr;
  }
  const bool batched = b > 1;
  if (!batched) {
    p.items = (long long)sh.S * sh.RQ;
  } else {
    const int rbq = kWarps * batched_qpw(p);
    p.items = (long long)sh.S * ((sh.RQ + rbq - 1) / rbq);
  }
  int grid = (int)std::min<long long>((long long)num_sms(), p.items);
  // fused mode (b = 1): whole slices per CTA group, S*J CTAs with J per slice,
  // when that idles at most 8 % of the SMs; the reduction then runs in-kernel
  p.fused_J = 0;
  if (!batched && p.xmode != 4) {
    const int sms = num_sms();
    const int J = sh.S <= sms ? sms / sh.S : 0;
    if (J >= 1 && J <= kFusedMaxJ && sh.S <= kFusedMaxJ && sh.S * J * 100 >= sms * 92 && sh.RQ >= J) {
      p.fused_J = J;
      grid = sh.S * J;
    }
  }
  cudaError_t e = sh.has_z ? dispatch_q<true>(p, grid, st, batched) : dispatch_q<false>(p, grid, st, batched);
  if (e != cudaSuccess) return e;
  if (p.fused_J > 0) return cudaSuccess;  // reduced in-kernel
  if (p.xmode == 2) return cudaSuccess;  // experiment: no reduction (wrong results, timing only)
  return launch_reduce(p, st);
}

}  // namespace lg
