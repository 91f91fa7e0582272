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
// ---------------------------------------------------------------------------
// Tensor-parallel exchange fused into the GEMV epilogue (NEXT-1, lutgemm_p2p.cu).
// Runs in the R reducer CTAs of every row-quad group after the group's slice partials are
// complete; reducer (fj, ri) owns rows [r0, r1) (a share of the group's 8-row units; every rank
// runs the same partition, so the same reducer on another rank owns the same rows), one thread
// per row, the S slice partials summed in slice order NS per L2 round trip (R11).
//   rows (p2p_mode 1, m-split): y[yoff + r] locally; (r, r+1) as one half2 LL word into every
//     peer's window; then the peers' rows r of their shards out of the local window into y.
//   cols (p2p_mode 2, n-split): reduce-scatter + all-gather.  The fp32 row sum goes as an LL
//     word to the owner o = r / mb, slot [self]; on the owner the same reducer share sums its
//     owned rows over the P slots in rank order (deterministic, identical on every rank), rounds
//     to fp16 and sends (r, r+1) half2 LL words to every peer; the other owners' rows are read
//     out of the local window.
// LL ("low-latency") words: 8 bytes = data | stamp << 32, written and read as ONE aligned 64-bit
// access (single-copy atomic), so a reader that sees the round's stamp sees the data -- no fence,
// no separate signal, no barrier on the path (the protocol NCCL uses for small messages).
// stamp = low 32 bits of round + 1; the window is double-buffered by round parity, so a stale
// word of the same parity carries stamp - 2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_ll(uint8_t* p, uint32_t d, uint32_t stamp) {
  const unsigned long long w = ((unsigned long long)stamp << 32) | d;
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
// a peer that never writes (crashed, or a call sequence that differs between ranks) must not hang
// the GPU: after timeout_ns without the round's word the kernel traps (the launch fails loudly)
__device__ __forceinline__ uint32_t ld_ll(const uint8_t* p, uint32_t stamp, unsigned long long timeout_ns) {
  unsigned long long w;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  if ((uint32_t)(w >> 32) != stamp) {
    const unsigned long long t0 = globaltimer_ns();
    do {
      __nanosleep(16);
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
      if (globaltimer_ns() - t0 > timeout_ns) __trap();
    } while ((uint32_t)(w >> 32) != stamp);
  }
  return (uint32_t)w;
}

// row r of the result: the S slice partials summed in slice order, NS per L2 round trip
template <int NS>
__device__ __forceinline__ float row_sum(const KParams& p, int r) {
  float v = 0.f;
  const float* pp = p.partial + r;
  for (int ss0 = 0; ss0 < p.sh.S; ss0 += NS) {
    float t[NS];
#pragma unroll
    for (int kk = 0; kk < NS; ++kk) t[kk] = (ss0 + kk < p.sh.S) ? __ldcg(pp + (size_t)(ss0 + kk) * p.sh.m4) : 0.f;
#pragma unroll
    for (int kk = 0; kk < NS; ++kk)
      if (ss0 + kk < p.sh.S) v += t[kk];
  }
  return v;
}

// fp16 of this lane's row (low half) and of the next lane's row (high half): the LL payload
__device__ __forceinline__ uint32_t half2_word(__half h) {
  const uint32_t hb = (uint32_t)__half_as_ushort(h);
  const uint32_t hn = __shfl_xor_sync(kFull, hb, 1);
  return hb | (hn << 16);
}

// The round: every CTA's thread 0 reads it right after the PDL wait (the previous call is complete:
// a relaxed load suffices) and counts in with a release RMW -- neither result is waited for until
// the main loop is over, so nothing stalls the LUT build.  After its main loop the CTA that counted
// in last (every CTA had read the round before counting in) acquires and advances it; the next
// call reads it after its own PDL wait.  The reducers take the round from shared memory.
template <int NS>
__device__ __forceinline__ void p2p_epilogue(const KParams& p, unsigned long long round, int R, int ri, int g0,
                                             int g1) {
  const Shape& sh = p.sh;
  const int P = p.npeers, self = p.p2p_self, tid = (int)threadIdx.x, lane = tid & 31;
  const int par = (int)(round & 1ull);
  const uint32_t stamp = (uint32_t)(round + 1ull);
  uint8_t* const mine = p.p2p_win[par][self];
  const int u0g = g0 / 2, u1g = (g1 + 1) / 2;  // the group's 8-row units (groups start on even quads)
  const int r0 = 8 * (u0g + (int)((long long)(u1g - u0g) * ri / R));
  const int r1 = min(sh.m, 8 * (u0g + (int)((long long)(u1g - u0g) * (ri + 1) / R)));
  // warp-uniform loops (the half2 pairing shuffles): row r = base + lane, base even
  if (p.p2p_mode == 1) {
    const int ms = sh.m;  // ms % 8 == 0 (host-checked): row pairs never straddle a shard
    for (int base = r0 + (tid & ~31); base < r1; base += kThreads) {
      const int r = base + lane;
      const bool ok = r < r1;
      const __half h = __float2half_rn(ok ? row_sum<NS>(p, r) : 0.f);
      if (ok) p.y[p.yoff + r] = h;
      const uint32_t word = half2_word(h);
      if (ok && !(lane & 1))
        for (int pr = 0; pr < P; ++pr)
          if (pr != self) st_ll(p.p2p_win[par][pr] + 4 * (size_t)(p.yoff + r), word, stamp);
    }
    for (int base = r0 + (tid & ~31); base < r1; base += kThreads) {
      const int r = base + lane;
      if (r < r1 && !(lane & 1))
        for (int k = 0; k < P - 1; ++k) {
          const int pr = k + (k >= self ? 1 : 0), rr = pr * ms + r;
          const uint32_t w = ld_ll(mine + 4 * (size_t)rr, stamp, p.p2p_timeout_ns);
          p.y[rr] = __ushort_as_half((unsigned short)(w & 0xFFFFu));
          p.y[rr + 1] = __ushort_as_half((unsigned short)(w >> 16));
        }
    }
  } else {
    const int m = sh.m, mb = p.p2p_mb;
    // each fp32 row to its owner's slot [self]; on the owner the same thread sums its owned rows
    // over the P slots in rank order (its own slot's value straight from the register), rounds to
    // fp16 and sends the row pairs to every peer.  Every rank sends an iteration's rows before it
    // waits for that iteration's words, so the waits cannot deadlock.
    for (int base = r0 + (tid & ~31); base < r1; base += kThreads) {
      const int r = base + lane;
      const bool ok = r < r1;
      const float v = ok ? row_sum<NS>(p, r) : 0.f;
      const int o = r / mb;
      const bool own = ok && o == self;
      if (ok && !own) st_ll(p.p2p_win[par][o] + 8 * ((size_t)self * mb + (r - o * mb)), __float_as_uint(v), stamp);
      float sum = 0.f;
      if (own)
        for (int pr = 0; pr < P; ++pr)
          sum += pr == self ? v : __uint_as_float(ld_ll(mine + 8 * ((size_t)pr * mb + (r - o * mb)), stamp, p.p2p_timeout_ns));
      const __half h = __float2half_rn(sum);
      if (own) p.y[r] = h;
      if (P > 1) {
        const uint32_t word = half2_word(h);
        if (own && !(lane & 1))
          for (int pr = 0; pr < P; ++pr)
            if (pr != self) st_ll(p.p2p_win[par][pr] + p.p2p_yarea + 4 * (size_t)r, word, stamp);
      }
    }
    // the other owners' rows of this share, out of the local window
    if (P > 1)
      for (int base = r0 + (tid & ~31); base < r1; base += kThreads) {
        const int r = base + lane;
        if (r < r1 && !(lane & 1) && r / mb != self) {
          const uint32_t w = ld_ll(mine + p.p2p_yarea + 4 * (size_t)r, stamp, p.p2p_timeout_ns);
          p.y[r] = __ushort_as_half((unsigned short)(w & 0xFFFFu));
          if (r + 1 < m) p.y[r + 1] = __ushort_as_half((unsigned short)(w >> 16));
        }
      }
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

  unsigned long long p2p_rd = 0;  // EP: the round (thread 0) and its count-in rank
  unsigned p2p_k = 0;
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
      if (EP && tid == 0) {
        p2p_rd = ld_relaxed_u64(p.p2p_round);
        p2p_k = atom_add_release_u32(p.counters + 2 * kFusedMaxJ + 2, 1u);
      }
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
    if (EP && tid == 0) {
      *reinterpret_cast<unsigned long long*>(sm.misc_p + kMiscRound) = p2p_rd;
      if (p2p_k == gridDim.x - 1) {  // the last to count in: every CTA has read the round
        unsigned* rcnt = p.counters + 2 * kFusedMaxJ + 2;
        fence_acq_rel_gpu();
        *rcnt = 0u;
        *reinterpret_cast<volatile unsigned long long*>(const_cast<unsigned long long*>(p.p2p_round)) = p2p_rd + 1ull;
      }
    }
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
      const unsigned long long round = *reinterpret_cast<const unsigned long long*>(sm.misc_p + kMiscRound);
      if (sh.S <= 16) p2p_epilogue<16>(p, round, R, ri, g0, g1);
      else p2p_epilogue<48>(p, round, R, ri, g0, g1);
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
