// gemv_kernel.cuh -- the sm_100a LUT-GEMV kernel template (b = 1), instantiated per MODE by
// lutgemm_gemv.cu (plain) and lutgemm_gemv_ep.cu (fused TP epilogue), compiled in parallel.
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
//  * after the programmatic-dependent-launch wait each thread loads its 8 x
//    values from L2 straight into registers for the LUT build (the bulk-copy
//    staging into shared memory remains as LUTGEMM_XDIRECT=0);
//  * lookups summed and scaled with packed f32x2 adds/FMAs (FADD2/FFMA2),
//    two rows per instruction;
//  * per-row partials reduced across lanes by a 6-shuffle transpose-reduce and
//    written to an fp32 split-K workspace; the cross-slice sum runs in the same
//    kernel (arrival-ordered on a self-resetting counter, fixed slice order:
//    deterministic).  Batched products: lutgemm_smallb.cu, lutgemm_batched.cu.
#pragma once
#include "kernels_common.cuh"

namespace lg {

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
// 8 consecutive fp32 rows [r, r + 8) of the slice partials summed over the S slices in slice
// order (R11); rows >= m4 read as 0
__device__ __forceinline__ void sum8_rows(const float* partial, int S, int m4, int r, float (&v)[8]) {
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = 0.f;
  if (r + 8 <= m4) {
    for (int s = 0; s < S; ++s) {
      const float4 a = __ldcg(reinterpret_cast<const float4*>(partial + (size_t)s * m4 + r));
      const float4 b = __ldcg(reinterpret_cast<const float4*>(partial + (size_t)s * m4 + r + 4));
      v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
      v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
    }
  } else {
    for (int s = 0; s < S; ++s)
      for (int k = 0; k < 8 && r + k < m4; ++k) v[k] += __ldcg(partial + (size_t)s * m4 + r + k);
  }
}

// ---------------------------------------------------------------------------
// Tensor-parallel exchange fused into the GEMV epilogue (NEXT-1, lutgemm_p2p.cu).
// Runs in the R reducer CTAs of every row-quad group (NRED = J R CTAs, all resident), after the
// group's slice partials are complete.  Rows of 8-row units [8u, 8u + 8), 16-byte stores.
//   rows (p2p_mode 1, m-split):  fp16 rows of this rank's shard -> this rank's y (local) and every
//     peer's window[par] at row yoff + r; signal A; wait for the P signals A; copy the peers' rows
//     out of the local window into y.
//   cols (p2p_mode 2, n-split):  fp32 partial rows -> the owner's window[par] slot [self]
//     (reduce-scatter); signal A; wait; sum the owned block over the P slots in rank order
//     (deterministic), fp16 -> y (local) and every peer's window y-area; signal B; wait; copy the
//     peers' blocks out of the local window into y.
// Signals: the grid's last CTA through a phase (acq_rel counter, gpu scope) issues
// fence.acq_rel.sys and red.release.sys.u64 on every rank's counter; waits are ld.acquire.sys by
// thread 0 followed by a CTA barrier (the chain: stores -> bar.sync -> acq_rel RMW -> last CTA's
// acquire -> fence.sys -> release to the peer -> the peer's acquire -> its bar.sync -> its loads).
// The last CTA of the final phase advances the device-side round (parity of the double buffer).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 pack_half8(const float (&v)[8]) {
  uint4 h;
  h.x = pack_half2(v[0], v[1]);
  h.y = pack_half2(v[2], v[3]);
  h.z = pack_half2(v[4], v[5]);
  h.w = pack_half2(v[6], v[7]);
  return h;
}

// store `cnt` (<= 8) fp16 values of h at dst (16-byte store when whole)
__device__ __forceinline__ void store_half8(uint8_t* dst, const uint4& h, int cnt) {
  if (cnt >= 8) {
    *reinterpret_cast<uint4*>(dst) = h;
  } else {
    const uint16_t* hs = reinterpret_cast<const uint16_t*>(&h);
    for (int k = 0; k < cnt; ++k) reinterpret_cast<uint16_t*>(dst)[k] = hs[k];
  }
}

// grid-wide phase barrier of the NRED reducer CTAs: the last to arrive (resetting the counter)
// runs `last` in thread 0; then every CTA waits until its own signal counter reaches `target`
template <typename F>
__device__ __forceinline__ void p2p_phase(unsigned* cnt, unsigned nred, const unsigned long long* my_sig,
                                          unsigned long long target, F last) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atom_add_acq_rel_u32(cnt, 1u) == nred - 1) {
      *cnt = 0u;
      last();
    }
    while (ld_acquire_sys_u64(my_sig) < target) __nanosleep(32);
  }
  __syncthreads();
}

// copy units [u0, u1) of 8 fp16 rows from src to dst (both indexed from row 0), rows < rows_end
__device__ __forceinline__ void copy_rows(__half* dst, const uint8_t* src, int u0, int u1, int rows_end) {
  for (int u = u0 + (int)threadIdx.x; u < u1; u += kThreads) {
    const int r = 8 * u;
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(src) + u);
    store_half8(reinterpret_cast<uint8_t*>(dst + r), v, rows_end - r);
  }
}

__device__ __forceinline__ void p2p_epilogue(const KParams& p, int J, int R, int fj, int ri, int g0, int g1) {
  const Shape& sh = p.sh;
  const int P = p.npeers, self = p.p2p_self;
  const unsigned nred = (unsigned)(J * R);
  const int red = fj * R + ri;  // this CTA's index among the reducers
  unsigned* cnt = p.counters + 2 * kFusedMaxJ;  // 3 phase counters
  const unsigned long long round = ld_acquire_u64(p.p2p_round);  // previous round complete (PDL wait)
  const int par = (int)(round & 1ull);
  const unsigned long long target = (round + 1ull) * (unsigned long long)P;
  unsigned long long* const* sig = p.p2p_sig;  // sig[pr][0] = A, [1] = B, [2] = round (self only)
  auto signal_all = [&](int which) {
    fence_acq_rel_sys();
    for (int pr = 0; pr < P; ++pr) red_release_sys_add_u64(sig[pr] + which, 1ull);
  };
  const int u0g = g0 / 2, u1g = (g1 + 1) / 2;  // the group's 8-row units (groups start on even quads)
  const int u0 = u0g + (int)((long long)(u1g - u0g) * ri / R), u1 = u0g + (int)((long long)(u1g - u0g) * (ri + 1) / R);
  auto share = [&](int units, int& a, int& b) {  // this reducer's share of `units` work units
    a = (int)((long long)units * red / nred);
    b = (int)((long long)units * (red + 1) / nred);
  };
  if (p.p2p_mode == 1) {
    const int ms = sh.m;
    for (int u = u0 + (int)threadIdx.x; u < u1; u += kThreads) {
      const int r = 8 * u;
      float v[8];
      sum8_rows(p.partial, sh.S, sh.m4, r, v);
      const uint4 h = pack_half8(v);
      store_half8(reinterpret_cast<uint8_t*>(p.y + p.yoff + r), h, ms - r);
      const size_t off = 2 * (size_t)(p.yoff + r);
      for (int pr = 0; pr < P; ++pr)
        if (pr != self) store_half8(p.p2p_win[par][pr] + off, h, ms - r);
    }
    p2p_phase(cnt, nred, sig[self], target, [&] { signal_all(0); });
    // the peers' rows: (P - 1) ms rows out of the local window
    const int upr = ms / 8;  // ms % 8 == 0 (checked on the host)
    int a, b;
    share((P - 1) * upr, a, b);
    for (int w = a + (int)threadIdx.x; w < b; w += kThreads) {
      const int k = w / upr, pr = k + (k >= self ? 1 : 0), u = pr * upr + w % upr;
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p.p2p_win[par][self]) + u);
      *reinterpret_cast<uint4*>(p.y + 8 * u) = v;
    }
  } else {
    const int m = sh.m, mb = p.p2p_mb;
    for (int u = u0 + (int)threadIdx.x; u < u1; u += kThreads) {
      const int r = 8 * u;
      float v[8];
      sum8_rows(p.partial, sh.S, sh.m4, r, v);
      const int o = r / mb;
      float* dst = reinterpret_cast<float*>(p.p2p_win[par][o]) + (size_t)self * mb + (r - o * mb);
      if (r + 8 <= m) {
        reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
      } else {
        for (int k = 0; k < m - r; ++k) dst[k] = v[k];
      }
    }
    p2p_phase(cnt, nred, sig[self], target, [&] { signal_all(0); });
    // owned block [self mb, self mb + mb): sum the P slots in rank order, fp16 -> y and every peer
    const float* slots = reinterpret_cast<const float*>(p.p2p_win[par][self]);
    const int b0 = self * mb, rows = max(0, min(mb, m - b0));
    int a, b;
    share((rows + 7) / 8, a, b);
    for (int w = a + (int)threadIdx.x; w < b; w += kThreads) {
      const int lr = 8 * w;
      float v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = 0.f;
      for (int pr = 0; pr < P; ++pr) {
        const float4 x0 = __ldcg(reinterpret_cast<const float4*>(slots + (size_t)pr * mb + lr));
        const float4 x1 = __ldcg(reinterpret_cast<const float4*>(slots + (size_t)pr * mb + lr + 4));
        v[0] += x0.x; v[1] += x0.y; v[2] += x0.z; v[3] += x0.w;
        v[4] += x1.x; v[5] += x1.y; v[6] += x1.z; v[7] += x1.w;
      }
      const uint4 h = pack_half8(v);
      store_half8(reinterpret_cast<uint8_t*>(p.y + b0 + lr), h, rows - lr);
      const size_t off = p.p2p_yarea + 2 * (size_t)(b0 + lr);
      for (int pr = 0; pr < P; ++pr)
        if (pr != self) store_half8(p.p2p_win[par][pr] + off, h, rows - lr);
    }
    if (P > 1) {
      p2p_phase(cnt + 1, nred, sig[self] + 1, target, [&] { signal_all(1); });
      // the peers' blocks out of the local window
      const int ub = mb / 8;
      share((P - 1) * ub, a, b);
      for (int w = a + (int)threadIdx.x; w < b; w += kThreads) {
        const int k = w / ub, pr = k + (k >= self ? 1 : 0), lu = w % ub;
        const int r = pr * mb + 8 * lu;
        if (r >= m) continue;
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p.p2p_win[par][self] + p.p2p_yarea) + r / 8);
        store_half8(reinterpret_cast<uint8_t*>(p.y + r), v, m - r);
      }
    }
  }
  // the last reducer to finish advances the round: every reducer has read it by now
  __syncthreads();
  if (threadIdx.x == 0 && atom_add_acq_rel_u32(cnt + 2, 1u) == nred - 1) {
    cnt[2] = 0u;
    *reinterpret_cast<volatile unsigned long long*>(p.p2p_sig[self] + 2) = round + 1ull;
  }
}

// MODE: 0 plain, 1 the fused tensor-parallel epilogue (EP).  Each mode is its own instantiation (and
// translation unit): the epilogue's code in the same function perturbs the main loop's register
// allocation (measured: +2 us on fc1 with the P2P epilogue inlined).
template <int QT, int ZM, int PD, int MODE>
__global__ void __launch_bounds__(kThreads, 1) lut_gemv_kernel(const KParams p) {
  constexpr bool EP = MODE == 1;
  constexpr bool HAS_Z = ZM != 0, CMP = ZM == 2;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(kFull, tid >> 5, 0);  // warp-uniform for the compiler
  const Shape sh = p.sh;
  const int q = QT <= 4 ? QT : sh.q;
  const bool cg = QT == 8 && sh.gcls == kGrpChunk;  // per-chunk scales (ring_compute_cg)
  const int J = p.fused_J;
  long long it0, it1;
  int fs = 0, fj = 0;  // fused mode: this CTA's slice and row group
  if (J > 0) {
    fused_slot(p, fs, fj);
    it0 = (long long)fs * sh.RQ + p.gq[fj];
    it1 = (long long)fs * sh.RQ + p.gq[fj + 1];
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

  const SmemMap sm = map_smem(smem, p.smem_bytes > 0 ? p.smem_bytes : kSmemBytesBase);
  __half* xbuf0 = reinterpret_cast<__half*>(sm.misc_p);
  __half* xbuf1 = reinterpret_cast<__half*>(sm.misc_p + 2048);
  const uint32_t bar0 = sm.misc + 4096, bar1 = sm.misc + 4104;
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)(4 * lane + 128) << 8) | (uint32_t)(4 * lane);
  if (!p.xdirect) {  // the bulk-copy staging of x needs its mbarriers (direct mode: no barrier here)
    if (tid == 0) {
      mbar_init(bar0, 1);
      mbar_init(bar1, 1);
      fence_mbar_init();
    }
    __syncthreads();
  }

  constexpr int NB = PD + 1;  // ring of quad buffers: the load of quad t + PD is issued before quad t is computed
  int e = 0;
  long long it = it0;
  while (it < it1) {
    // the segment: slice s, row quads [rq_a, rq_b) (fused mode: one segment, no 64-bit division)
    int s, rq_a, rq_b;
    if (J > 0) {
      s = fs;
      rq_a = p.gq[fj];
      rq_b = p.gq[fj + 1];
    } else {
      s = (int)(it / sh.RQ);
      rq_a = (int)(it - (long long)s * sh.RQ);
      rq_b = (int)min((long long)sh.RQ, (long long)rq_a + (it1 - it));
    }
    const long long itn = it + (rq_b - rq_a);
    const int Ls = slice_lanes(sh.n, s);
    const bool lane_ok = lane < Ls;
    const LaneAddr la = lane_addr(sh, p.fs, p.data, s, Ls, lane_ok ? lane : 0);
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
    // load quad tl of the warp into b (keys, scales, z)
    auto load_quad = [&](Ring<QT>& b) {
      if (nt == 0) return;  // a warp without quads in the segment loads nothing
#pragma unroll
      for (int i = 0; i < QT; ++i)
        if (QT <= 4 || i < q) b.k[i] = ldg_stream_u4(lk + i * la.kstride);
      if (QT == 8) {
        b.ap = lal;
        b.zp = lz;
      }
      if (!cg) {
#pragma unroll
        for (int i = 0; i < QT; ++i)
          if ((QT <= 4 || i < q) && (!CMP || i == 0)) b.a[i] = ldg_nc_u2(lal + 8 * i);
        if (HAS_Z) b.z = ldg_nc_u2(lz);
      }
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
      if (trace) trace[3] = globaltimer_ns();
      if (warp == 0 && !p.xdirect)
        stage_x(xbuf0, bar0, p.x, sh.n, s * kSliceCols, slice_cols(sh.n, s), 32, 1, 1, lane);
    }
    // this thread's 8 x values of slice s for the LUT build: direct mode loads them from global
    // memory (L2) into registers, no shared-memory staging, mbarrier or barrier on the path
    const int xc = (4 * lane + (warp & 3)) * 8;  // column of the chunk within the slice
    uint4 xraw = make_uint4(0, 0, 0, 0);
    if (p.xdirect && xc < slice_cols(sh.n, s)) {
      xraw = ldcg_u4(p.x + (size_t)s * kSliceCols + xc);
    }
    if (e > 0 || J == 0) {
#pragma unroll
      for (int d = 0; d < PD; ++d) load_quad(buf[d]);
    }
    // 2. (bulk-copy mode) wait for the staged x slice; build the 128 LUTs of the slice
    if (!p.xdirect) {
      if (e == 0) __syncthreads();  // the zero-fill of the x buffer is visible
      mbar_wait((e & 1) ? bar1 : bar0, (uint32_t)((e >> 1) & 1));
      xraw = *reinterpret_cast<const uint4*>(((e & 1) ? xbuf1 : xbuf0) + xc);
    }
    if (trace && e == 0) trace[1] = globaltimer_ns();
    build_table_part(sm.lut + table_offset(lane, warp & 3), xraw, warp >> 2);
    __syncthreads();
    if (trace && e == 0) trace[2] = globaltimer_ns();
    // 3. stage the next segment's x slice into the other buffer
    if (warp == 0 && itn < it1 && !p.xdirect) {
      const int sn = (int)(itn / sh.RQ);
      stage_x((e & 1) ? xbuf0 : xbuf1, (e & 1) ? bar0 : bar1, p.x, sh.n, sn * kSliceCols,
              slice_cols(sh.n, sn), 32, 1, 1, lane);
    }
    const float xsum = (HAS_Z && lane_ok && !cg) ? lane_xsum(sm.lut, lane) : 0.f;
    float xs4[4] = {0.f, 0.f, 0.f, 0.f};  // chunk-group shapes: x sum of each of the lane's chunks
    if (QT == 8 && HAS_Z && cg && lane_ok) {
#pragma unroll
      for (int j = 0; j < 4; ++j) xs4[j] = lds_f32<0>(sm.lut + table_offset(lane, j) + 255u * 256u);
    }
    // 4. main loop: per quad and plane 16 PRMT + 16 LDS + 6 FADD2 + 2 FFMA2, then
    //    a 6-shuffle transpose-reduce and one store per row of the slice partial
    float* pw = p.partial + (size_t)s * sh.m4 + 4 * (rq_a + warp) + (lane >> 3);  // this warp's next partial
    auto quad = [&](const Ring<QT>& b) {
      f32x2 acc01, acc23;
      if constexpr (QT == 8) {
        if (cg) ring_compute_cg<HAS_Z>(b, lc, xs4, acc01, acc23, q);
        else ring_compute<QT, ZM>(b, lc, xsum, acc01, acc23, q);
      } else {
        ring_compute<QT, ZM>(b, lc, xsum, acc01, acc23, q);
      }
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
    unsigned& s_k = *reinterpret_cast<unsigned*>(sm.misc_p + kMiscArrive);  // no static shared memory
    const int R = max(1, min(p.reducers, sh.S));
    // Arrival: a wrapping counter (atom.inc, back to 0 after the S-th arrival: no reset step, no
    // departure atomic on the way out).  Release: the CTA's partial stores (ordered before by the
    // barrier) are visible to whoever acquires the count.
    unsigned* arrive = p.counters + fj;
    __syncthreads();  // all partial stores of this CTA are issued
    if (tid == 0) {
      // wrapping arrival counter: k = arrivals before this one; it returns to 0 with the S-th, so a
      // reducer that is not last waits until the counter falls to <= k (acquire: synchronizes with
      // the last arriver's RMW, which acquired every earlier arrival's partial stores)
      const unsigned kk = atom_inc_acq_rel_u32(arrive, (unsigned)sh.S - 1u);
      if (kk >= (unsigned)(sh.S - R) && kk != (unsigned)sh.S - 1u)
        while (ld_acquire_u32(arrive) > kk) __nanosleep(32);
      s_k = kk;
    }
    __syncthreads();
    const int k = (int)s_k;
    if (k < sh.S - R) return;
    if (trace) trace[5] = globaltimer_ns();  // (re-used) the group is complete
    const int ri = k - (sh.S - R);
    const int g0 = p.gq[fj], g1 = p.gq[fj + 1];
    if (!EP) {
      // plain output: this reducer's rows of the group, one thread per row
      const int r0 = 4 * (g0 + (int)((long long)(g1 - g0) * ri / R));
      const int r1 = min(sh.m, 4 * (g0 + (int)((long long)(g1 - g0) * (ri + 1) / R)));
      // sum over the S slices in slice order, up to NS slices per L2 round trip (16, or 48 for the
      // wide layers: fc2 has S = 48; a 48-wide batch measured slower for S = 12)
      auto reduce_rows = [&](auto ns) {
        constexpr int NS = decltype(ns)::value;
        for (int r = r0 + tid; r < r1; r += kThreads) {
          float v = 0.f;
          const float* pp = p.partial + r;
          for (int ss0 = 0; ss0 < sh.S; ss0 += NS) {
            float t[NS];
#pragma unroll
            for (int kk = 0; kk < NS; ++kk) t[kk] = (ss0 + kk < sh.S) ? __ldcg(pp + (size_t)(ss0 + kk) * sh.m4) : 0.f;
#pragma unroll
            for (int kk = 0; kk < NS; ++kk)
              if (ss0 + kk < sh.S) v += t[kk];
          }
          if (p.yf) p.yf[r] = v;
          else p.y[r] = __float2half_rn(v);
        }
      };
      if (sh.S <= 16) reduce_rows(std::integral_constant<int, 16>{});
      else reduce_rows(std::integral_constant<int, 48>{});
    } else {
      p2p_epilogue(p, J, R, fj, ri, g0, g1);
    }
    if (trace) trace[6] = globaltimer_ns();  // reduction share done
    return;
  }
  pdl_launch_dependents();  // the reduction kernel may now be scheduled
}

// launcher of the MODE instantiations (dispatch on q and the scale format)
template <int MODE>
struct GemvLaunchMode {
  template <int QT, int ZM>
  struct F {
    static cudaError_t run(const KParams& p, int grid, cudaStream_t st) {
      // quads in flight per warp while one is computed (ring of PD + 1 buffers)
      constexpr int PD = QT <= 1 ? 6 : (QT <= 2 ? 4 : (QT <= 4 ? 2 : 1));
      return launch(lut_gemv_kernel<QT, ZM, PD, MODE>, grid, p, st);
    }
  };
};

cudaError_t launch_gemv_ep(const KParams& p, int grid, cudaStream_t st);  // lutgemm_gemv_ep.cu

}  // namespace lg
