// lutgemm_batched.cu -- the vector-slot batched LUT-GEMM (b > 4; 2 <= b <= 4 on
// request) and its cross-slice reduction kernel.  Method and design: the
// section comment below, lutgemm_gemv.cu and DESIGN.md.
#include <algorithm>
#include <cstdlib>

#include "kernels_common.cuh"

namespace lg {

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
  const bool cg = QT == 8 && sh.gcls == kGrpChunk;  // per-chunk scales (vring_compute_cg)
  const int NV = p.nv, NW = LR / NV, bpad = V * NV, b = p.b, spi = p.spi;
  const int qi = lane / LR, wv = lane % LR, w = wv / NV, v = wv % NV;
  const int rbq = (NTH / 32) * QPW;  // row quads per work item
  const int NRB = (sh.RQ + rbq - 1) / rbq;
  const int it0 = (int)(p.items * blockIdx.x / gridDim.x);
  const int it1 = (int)(p.items * (blockIdx.x + 1) / gridDim.x);
  if (it0 >= it1) return;

  const SmemMap sm = map_smem(smem, p.smem_bytes > 0 ? p.smem_bytes : kSmemBytesBase);
  const __half* xtile0 = reinterpret_cast<const __half*>(sm.misc_p);
  const __half* xtile1 = reinterpret_cast<const __half*>(sm.misc_p + 2048);
  const uint32_t xt0 = sm.misc, xt1 = sm.misc + 2048;
  const uint32_t lc = (sm.lut & 0xFFFF0000u) | ((uint32_t)((LR + wv) * 4 * V) << 8) | (uint32_t)(wv * 4 * V);

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
      const int per_row = 4 * NW;  // 16-byte cells per tile row
      const int bt = tid / per_row, c = tid % per_row;
      const bool ok = bt < b && 32 * st.k * NW + 8 * c < slice_cols(sh.n, st.s);  // zero past n
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
    const int k = lane_group(sh, st.s, pl);
    pt.aq = p.data + alpha_at(sh, st.s, Ls, rq, 0, k, 0);
    pt.zq = p.data + z_at(sh, st.s, Ls, rq, k, 0);
    return pt;
  };
  Ring<QT> ring[NB];
  VPtr nxt;  // pointers of the next step, positioned after its prologue groups
  bool nxt_ok;
  auto prologue = [&](const VStep& st) {
    const int rq_w = (st.it % NRB) * rbq + warp * QPW;
    nxt = lane_ptr(st, rq_w, nxt_ok);
#pragma unroll
    for (int d = 0; d < PD; ++d) vring_load<QT, ZM>(ring[d], nxt_ok && rq_w + V * d + qi < sh.RQ, nxt, q, cg);
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
      f32x2 xsJ[4][NP];                          // chunk-group shapes: per chunk
      if (QT == 8 && HAS_Z && cg) {
        vlut<V, 0>(0xFFFFFFFFu, lc, xsJ[0]);
        vlut<V, 1>(0xFFFFFFFFu, lc, xsJ[1]);
        vlut<V, 2>(0xFFFFFFFFu, lc, xsJ[2]);
        vlut<V, 3>(0xFFFFFFFFu, lc, xsJ[3]);
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (t + PD < NT) vring_load<QT, ZM>(ring[(t + PD) % NB], lane_ok && V * (t + PD) < nql, cur, q, cg);
        if constexpr (QT == 8) {
          if (cg) vring_compute_cg<V, HAS_Z>(ring[t % NB], lc, xsJ, acc[t], q);
          else vring_compute<V, QT, ZM>(ring[t % NB], lc, xs, acc[t], q);
        } else {
          vring_compute<V, QT, ZM>(ring[t % NB], lc, xs, acc[t], q);
        }
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


// V-wide slots (V = 2 only for b = 2); p.qpw = row quads per work item (256 or
// 128).  V = 2 runs 16 warps (128 registers: 4 rows x 2 batch x 16 quads of
// accumulators), V = 4 and q > 4 run 8 warps (255 registers).
template <int QT, int ZM>
struct BatchedLaunch {
  template <int V>
  static cudaError_t run_v(const KParams& p, int grid, cudaStream_t st) {
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
  static cudaError_t run(const KParams& p, int grid, cudaStream_t st) {
    return p.b == 2 ? run_v<2>(p, grid, st) : run_v<4>(p, grid, st);
  }
};

cudaError_t launch_batched(const KParams& p, int grid, cudaStream_t st) {
  return dispatch_qz<BatchedLaunch>(p, grid, st);
}

cudaError_t launch_reduce_batched(const KParams& p, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.sh.m4 + 63) / 64);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = const_cast<cudaLaunchAttribute*>(pdl_attr());
  cfg.numAttrs = 1;
  const int S2 = (p.sh.S + p.spi - 1) / p.spi;
  return cudaLaunchKernelEx(&cfg, lut_reduce_batched_kernel, (const float*)p.partial, S2, p.b, 1 << p.bl, p.sh.m,
                            p.sh.m4, p.y, p.yf);
}

// Work split of the batched kernel: items = (range of spi slices, row block of
// rbq = 256 or 128 quads); pick (rbq, spi) minimising waves * spi * (per-sub-
// slice lookup time + LUT rebuild time), ties to fewer partials (larger spi).
void plan_batched(const Shape& sh, int sms, KParams& p) {
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

}  // namespace lg
