// lutgemm_smallb.cu -- 2 <= b <= 4 with the GEMV's streaming structure over
// sub-slices of 1024 / V columns (vector LUT slots of all V activation rows).
// Design: the section comment in kernels_common.cuh and DESIGN.md.
#include "kernels_common.cuh"

namespace lg {

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
  int fs = 0, fj = 0;  // fused mode: this CTA's sub-slice and quad-group range
  if (J > 0) {
    fused_slot(p, fs, fj);
    it0 = (long long)fs * NG + p.gq[fj];
    it1 = (long long)fs * NG + p.gq[fj + 1];
  } else {
    it0 = p.items * blockIdx.x / gridDim.x;
    it1 = p.items * (blockIdx.x + 1) / gridDim.x;
  }
  if (it0 >= it1 && J == 0) return;
  if (J > 0) pdl_launch_dependents();

  const SmemMap sm = map_smem(smem, p.smem_bytes > 0 ? p.smem_bytes : kSmemBytesBase);
  const uint32_t xt0 = sm.misc, xt1 = sm.misc + 2048;
  const __half* xtile0 = reinterpret_cast<const __half*>(sm.misc_p);
  const __half* xtile1 = reinterpret_cast<const __half*>(sm.misc_p + 2048);
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)((LR + w) * 4 * V) << 8) | (uint32_t)(w * 4 * V);
  // x tile of sub-slice hs: rows 0..V-1 of x (zero for rows >= b), 32 LR columns,
  // in the vector-slot cell order (xcell<V>, NV = 1)
  auto load_x = [&](uint32_t dst, int hs) {
    if (tid < 128) {
      const int s = hs / V, h = hs % V;
      const int per_row = 4 * LR;
      const int bt = tid / per_row, c = tid % per_row;
      const bool ok = bt < b && 32 * LR * h + 8 * c < slice_cols(sh.n, s);  // zero past n
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
    const LaneAddr la = lane_addr(sh, p.fs, p.data, s, Ls, LR * h + (lane_ok ? w : 0));
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
    unsigned& s_k = *reinterpret_cast<unsigned*>(sm.misc_p + kMiscArrive);  // no static shared memory
    const int R = max(1, min(p.reducers, SV));
    unsigned* arrive = p.counters + fj;  // wrapping arrival counter (see lut_gemv_kernel)
    __syncthreads();
    if (tid == 0) {
      // wrapping arrival counter: k = arrivals before this one; it returns to 0 with the S-th, so a
      // reducer that is not last waits until the counter falls to <= k (acquire: synchronizes with
      // the last arriver's RMW, which acquired every earlier arrival's partial stores)
      const unsigned kk = atom_inc_acq_rel_u32(arrive, (unsigned)SV - 1u);
      if (kk >= (unsigned)(SV - R) && kk != (unsigned)SV - 1u)
        while (ld_acquire_u32(arrive) > kk) __nanosleep(32);
      s_k = kk;
    }
    __syncthreads();
    const int k = (int)s_k;
    if (k < SV - R) return;
    const int ri = k - (SV - R);
    const int g0 = V * p.gq[fj], g1 = min(sh.RQ, V * p.gq[fj + 1]);
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
    return;
  }
  pdl_launch_dependents();
}


template <int QT, int ZM>
struct SmallbLaunch {
  static cudaError_t run(const KParams& p, int grid, cudaStream_t st) {
    constexpr int PD = QT <= 2 ? 3 : (QT <= 4 ? 2 : 1);
    if (p.b == 2) return launch(lut_gemvv_kernel<2, QT, ZM, PD>, grid, p, st);
    return launch(lut_gemvv_kernel<4, QT, ZM, PD>, grid, p, st);
  }
};

cudaError_t launch_smallb(const KParams& p, int grid, cudaStream_t st) {
  return dispatch_qz<SmallbLaunch>(p, grid, st);
}

}  // namespace lg
