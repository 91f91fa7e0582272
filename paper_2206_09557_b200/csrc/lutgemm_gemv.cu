// lutgemm_gemv.cu -- the sm_100a LUT-GEMV (b = 1) and the cross-slice reduction kernel.
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
      if (p.npeers > 0 && p.p2p_f32) {  // fused all-reduce: fp32 partial row into slot `rank` of every rank
        for (int pr = 0; pr < p.npeers; ++pr) reinterpret_cast<float*>(p.peer_y[pr])[p.yoff + r] = v;
      } else if (p.npeers > 0) {  // fused rows all-gather (NEXT-1): the row goes to every rank's output over NVLink
        const __half h = __float2half_rn(v);
        for (int pr = 0; pr < p.npeers; ++pr) p.peer_y[pr][p.yoff + r] = h;
      } else if (p.yf) {
        p.yf[r] = v;
      } else {
        p.y[r] = __float2half_rn(v);
      }
    }
    __syncthreads();
    if (tid == 0 && atomicAdd(depart, 1u) == (unsigned)R - 1) {  // the last reducer resets the pair
      *arrive = 0u;
      *depart = 0u;
    }
    if (p.npeers > 0 && tid == 0) {
      // The last reducer of the whole grid signals every rank.  Ordering of every
      // reducer's peer stores before that signal (PTX memory model, causality order
      // is transitive across scopes): stores -> bar.sync (CTA) -> this thread's
      // acq_rel RMW on `done` (gpu scope, both sides on this GPU) -> the last
      // reducer's acquiring RMW -> its fence.acq_rel.sys -> red.release.sys to the
      // peer -> the peer's ld.acquire.sys.  A system-scope fence in every reducer
      // (the first version) is not needed and cost 3.6 us per call.
      unsigned* done = p.counters + 2 * kFusedMaxJ;
      if (atom_add_acq_rel_u32(done, 1u) == (unsigned)(J * R) - 1) {
        *done = 0u;
        fence_acq_rel_sys();
        for (int pr = 0; pr < p.npeers; ++pr) red_release_sys_add_u32(p.peer_sig[pr], 1u);
        // ... and holds the grid open until every rank's rows of this round have
        // arrived here: the kernel's completion then means "gathered output ready"
        if (p.p2p_target) {
          while (ld_acquire_sys_u32(p.peer_sig[p.p2p_self]) < p.p2p_target) __nanosleep(64);
        }
      }
    }
    if (trace) trace[6] = globaltimer_ns();  // reduction share done
    return;
  }
  pdl_launch_dependents();  // the reduction kernel may now be scheduled
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


template <int QT, int ZM>
struct GemvLaunch {
  static cudaError_t run(const KParams& p, int grid, cudaStream_t st) {
    // quads in flight per warp while one is computed (ring of PD + 1 buffers)
    constexpr int PD = QT <= 1 ? 6 : (QT <= 2 ? 4 : (QT <= 4 ? 2 : 1));
    return launch(lut_gemv_kernel<QT, ZM, PD>, grid, p, st);
  }
};

cudaError_t launch_gemv(const KParams& p, int grid, cudaStream_t st) { return dispatch_qz<GemvLaunch>(p, grid, st); }

cudaError_t launch_reduce(const KParams& p, cudaStream_t st) {
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
  cfg.attrs = const_cast<cudaLaunchAttribute*>(pdl_attr());
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, lut_reduce_kernel, (const float*)p.partial, p.sh.S, p.b, p.sh.m, p.sh.m4, p.y,
                            p.yf);
}

// Fused all-reduce, local step: y[r] = sum over ranks pr = 0..P-1 (fixed order,
// deterministic) of slot[pr][r], fp16 round-to-nearest-even.  Launched with PDL
// behind the fused GEMV (which triggers its dependents early), so its CTAs are
// resident and waiting when the GEMV's last reducer has seen the round's signals.
__global__ void __launch_bounds__(256) p2p_sum_kernel(const float* __restrict__ slots, int P, int m,
                                                      __half* __restrict__ y) {
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  float v = __ldcg(slots + r);
  for (int pr = 1; pr < P; ++pr) v += __ldcg(slots + (size_t)pr * m + r);
  y[r] = __float2half_rn(v);
}

cudaError_t launch_p2p_sum(const float* slots, int P, int m, uint16_t* y, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  static bool attr_set = false;
  if (!attr_set) {  // same carveout as the GEMV: no L1/smem reconfiguration, co-resident while waiting
    cudaFuncSetAttribute(p2p_sum_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((m + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = const_cast<cudaLaunchAttribute*>(pdl_attr());
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, p2p_sum_kernel, slots, P, m, reinterpret_cast<__half*>(y));
}

}  // namespace lg
