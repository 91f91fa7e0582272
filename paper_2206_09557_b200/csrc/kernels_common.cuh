// kernels_common.cuh -- device helpers shared by the LUT-GEMM kernels
// (lutgemm_gemv.cu, lutgemm_batched.cu, lutgemm_smallb.cu) and the launch glue
// they share with lutgemm_dispatch.cu.  See lutgemm_gemv.cu for the method and
// DESIGN.md "Kernels" for the B200 design.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "layout.cuh"
#include "lutgemm_internal.h"
#include "ptx.cuh"

namespace lg {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMiscBytes = 8192;       // x double buffer (2 x 2 KB) + mbarriers + flags
// dynamic shared memory per CTA: the LUT (128 KB) on a 64 KB boundary + misc for any base alignment.
// The product kernels declare no static shared memory (tests/test_abi_cpu.py checks the SASS
// resource usage).  A 227 KB variant with a weight prefetch area before the PDL wait measured slower
// everywhere (measured and dropped): the larger carveout takes L1 capacity.
constexpr int kSmemBytesBase = 3 * 65536;
constexpr int kMiscArrive = 4128;      // misc-block offset of the fused reduction's arrival slot (u32)
constexpr int kMiscRound = 4136;       // misc-block offset of the P2P round read at kernel start (u64)
constexpr unsigned kFull = 0xffffffffu;

struct SmemMap {
  uint32_t lut;     // shared-window address of the LUT (multiple of 64 KB)
  uint32_t misc;    // shared-window address of the misc block
  uint8_t* misc_p;  // generic pointer to the misc block
};

__device__ __forceinline__ SmemMap map_smem(uint8_t* smem, int /*bytes*/) {
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
__device__ __forceinline__ void build_table_part(uint32_t tbl, uint4 raw, int h) {
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

// Stage x[beta][col0 .. col0 + nc) for beta < nb into buf[beta][0 .. 32*P)
// (fp16), zero-filling columns >= nc (nc % 8 == 0: whole 16-byte units) and
// batch rows nb..B-1.  Called by warp 0.
__device__ __forceinline__ void stage_x(__half* buf, uint32_t bar, const __half* x, int n, int col0, int nc,
                                        int P, int nb, int B, int lane) {
  const uint32_t bytes = (uint32_t)nc * 2u;
  if (lane == 0) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, bytes * (uint32_t)nb);
  }
  __syncwarp();
  if (lane < nb) bulk_g2s(smem_u32(buf + (size_t)lane * 32 * P), x + (size_t)lane * n + col0, bytes, bar);
  // zero-fill the rest (generic proxy, disjoint from the async writes)
  const int row_h = 32 * P;
  for (int beta = 0; beta < B; ++beta) {
    const int from = beta < nb ? nc : 0;
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
  const uint8_t* ap;  // chunk-group shapes (kGrpChunk, QT = 8 only): the quad's scale / z addresses,
  const uint8_t* zp;  // read at compute time (ring_compute_cg)
};

// Per-segment addressing of a lane's fields in the three slice regions.
struct LaneAddr {
  const uint8_t* kp;  // lane's key bytes of row quad 0, plane 0
  const uint8_t* ap;  // lane's alpha of row quad 0, plane 0
  const uint8_t* zp;  // lane's z of row quad 0
  uint32_t KB, AB, ZB;  // per-row-quad strides of the regions
  uint32_t kstride;     // bytes between planes of the key block (Ls * 16)
};

__device__ __forceinline__ LaneAddr lane_addr(const Shape& sh, const FullSlice& fs, const uint8_t* data, int s,
                                              int Ls, int lay) {
  LaneAddr a;
  const int k = lane_group(sh, s, lay);
  if (Ls == kLanesPerSlice) {  // full slice: host-computed constants (layout.cuh's formulas)
    const uint8_t* base = data + (size_t)s * fs.stride;
    const uint32_t qa = (uint32_t)scale_planes(sh);
    a.kp = base + (uint32_t)lay * 16u;
    a.ap = base + fs.aoff + (sh.gcls == kGrpChunk ? (uint32_t)lay * qa * 32u : (uint32_t)k * qa * 8u);
    a.zp = base + fs.zoff + (uint32_t)k * 8u;
    a.KB = fs.KB;
    a.AB = fs.AB;
    a.ZB = fs.ZB;
    a.kstride = kLanesPerSlice * 16u;
    return a;
  }
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

// Chunk-group shapes (g % 32 != 0, kGrpChunk; generic-q kernels only): every 8-column chunk of the
// lane's word has its own scale entry, so each lookup is scaled on its own:
//   acc[r] = sum_i sum_j alpha[r][chunk j][i] * T_{4l+j}[key_ij(r)]  (+ sum_j z[r][chunk j] * xsum_j)
// The scales (32 contiguous bytes per plane: chunks 0..3 x rows 0..3) and z are loaded here, not
// through the register ring: a correct, untuned path for the rare group sizes.
template <bool HAS_Z>
__device__ __forceinline__ void ring_compute_cg(const Ring<8>& r, uint32_t lc, const float (&xs)[4], f32x2& acc01,
                                                f32x2& acc23, int q) {
  acc01 = 0ull;
  acc23 = 0ull;
  for (int i = 0; i < q; ++i) {
    const uint4 A0 = ldg_nc_u4(r.ap + 32 * i), A1 = ldg_nc_u4(r.ap + 32 * i + 16);
    const uint4 w = r.k[i];
    acc01 = fma2(h2_to_f32x2(A0.x), pack2(lut1<0>(w.x, lc), lut1<0>(w.y, lc)), acc01);
    acc23 = fma2(h2_to_f32x2(A0.y), pack2(lut1<0>(w.z, lc), lut1<0>(w.w, lc)), acc23);
    acc01 = fma2(h2_to_f32x2(A0.z), pack2(lut1<1>(w.x, lc), lut1<1>(w.y, lc)), acc01);
    acc23 = fma2(h2_to_f32x2(A0.w), pack2(lut1<1>(w.z, lc), lut1<1>(w.w, lc)), acc23);
    acc01 = fma2(h2_to_f32x2(A1.x), pack2(lut1<2>(w.x, lc), lut1<2>(w.y, lc)), acc01);
    acc23 = fma2(h2_to_f32x2(A1.y), pack2(lut1<2>(w.z, lc), lut1<2>(w.w, lc)), acc23);
    acc01 = fma2(h2_to_f32x2(A1.z), pack2(lut1<3>(w.x, lc), lut1<3>(w.y, lc)), acc01);
    acc23 = fma2(h2_to_f32x2(A1.w), pack2(lut1<3>(w.z, lc), lut1<3>(w.w, lc)), acc23);
  }
  if (HAS_Z) {
    const uint4 Z0 = ldg_nc_u4(r.zp), Z1 = ldg_nc_u4(r.zp + 16);
    const uint32_t zc[8] = {Z0.x, Z0.y, Z0.z, Z0.w, Z1.x, Z1.y, Z1.z, Z1.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const f32x2 xx = pack2(xs[j], xs[j]);
      acc01 = fma2(h2_to_f32x2(zc[2 * j]), xx, acc01);
      acc23 = fma2(h2_to_f32x2(zc[2 * j + 1]), xx, acc23);
    }
  }
}

// sum of x over the lane's 32 columns = sum_j T_{4l+j}[255]
__device__ __forceinline__ float lane_xsum(uint32_t lut, int lane) {
  const uint32_t k255 = 255u * 256u;
  return (lds_f32<0>(lut + table_offset(lane, 0) + k255) + lds_f32<0>(lut + table_offset(lane, 1) + k255)) +
         (lds_f32<0>(lut + table_offset(lane, 2) + k255) + lds_f32<0>(lut + table_offset(lane, 3) + k255));
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
// 128 B); lane = qi * LR + wv, wv = w * NV + v: quad qi of a group of V
// consecutive row quads (all 4 rows of it), layout lane w of the sub-slice,
// batch vector v (rows vV..vV+V-1).
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
__device__ __forceinline__ void vring_load(Ring<QT>& r, bool ok, VPtr& pt, int q, bool cg = false) {
  constexpr bool HAS_Z = ZM != 0, CMP = ZM == 2;  // z term; compact scales (alpha_i = 2^(i-1) s)
  if (QT == 8) {  // chunk-group shapes read the scales at compute time (vring_compute_cg); null = skip
    r.ap = ok ? pt.aq : nullptr;
    r.zp = pt.zq;
  }
#pragma unroll
  for (int i = 0; i < QT; ++i) {
    if (QT <= 4 || i < q) {
      if (ok) {
        r.k[i] = ldg_stream_u4(pt.kq + i * pt.kstride);
        if (!cg) r.a[i] = (!CMP || i == 0) ? ldg_nc_u2(pt.aq + 8 * i) : make_uint2(0, 0);
      } else {
        r.k[i] = make_uint4(0, 0, 0, 0);
        r.a[i] = make_uint2(0, 0);
      }
    }
  }
  if (HAS_Z && !cg) r.z = ok ? ldg_nc_u2(pt.zq) : make_uint2(0, 0);
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

// chunk-group shapes (kGrpChunk, generic-q kernels): acc[rho][p] += sum_i sum_J alpha[rho][J][i] *
// (lookups of chunk J) + sum_J z[rho][J] * xs[J] -- each chunk of the lane's word scaled on its own
// (see ring_compute_cg); the scales are read here (32 contiguous bytes per plane)
template <int V, bool HAS_Z>
__device__ __forceinline__ void vring_compute_cg(const Ring<8>& r, uint32_t lc, const f32x2 (&xs)[4][V / 2],
                                                 f32x2 (&acc)[4][V / 2], int q) {
  constexpr int NP = V / 2;
  if (r.ap == nullptr) return;  // quad past the end
  for (int i = 0; i < q; ++i) {
    const uint4 A0 = ldg_nc_u4(r.ap + 32 * i), A1 = ldg_nc_u4(r.ap + 32 * i + 16);
    const uint32_t aw[8] = {A0.x, A0.y, A0.z, A0.w, A1.x, A1.y, A1.z, A1.w};  // chunk J: rows 01 = 2J, 23 = 2J+1
    const uint32_t kw[4] = {r.k[i].x, r.k[i].y, r.k[i].z, r.k[i].w};
#pragma unroll
    for (int rho = 0; rho < 4; ++rho) {
      f32x2 t[4][NP];
      vlut<V, 0>(kw[rho], lc, t[0]);
      vlut<V, 1>(kw[rho], lc, t[1]);
      vlut<V, 2>(kw[rho], lc, t[2]);
      vlut<V, 3>(kw[rho], lc, t[3]);
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        const float2 a = h2_to_f2(aw[2 * J + (rho >> 1)]);
        const float av = (rho & 1) ? a.y : a.x;
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) acc[rho][pp] = fma2(pack2(av, av), t[J][pp], acc[rho][pp]);
      }
    }
  }
  if (HAS_Z) {
    const uint4 Z0 = ldg_nc_u4(r.zp), Z1 = ldg_nc_u4(r.zp + 16);
    const uint32_t zw[8] = {Z0.x, Z0.y, Z0.z, Z0.w, Z1.x, Z1.y, Z1.z, Z1.w};
#pragma unroll
    for (int rho = 0; rho < 4; ++rho)
#pragma unroll
      for (int J = 0; J < 4; ++J) {
        const float2 zz = h2_to_f2(zw[2 * J + (rho >> 1)]);
        const float zv = (rho & 1) ? zz.y : zz.x;
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) acc[rho][pp] = fma2(pack2(zv, zv), xs[J][pp], acc[rho][pp]);
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
// ---------------------------------------------------------------------------
// b <= 4 with the GEMV's streaming structure.  With V = 2 (b = 2) or V = 4
// (b = 3, 4) a sub-slice of 1024 / V columns (layout lanes [LR h, LR h + LR) of a
// slice, LR = 32 / V; sub-slice hs = V s + h) holds the LUTs of all V
// activation rows: 4 LR chunks x 256 keys x V floats = 128 KB of vector slots
// (the batched kernel's slot layout with NV = 1), read with one PRMT + LDS.64 / LDS.128 per
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


// ---------------------------------------------------------------------------
// launch glue (lutgemm_dispatch.cu)
// ---------------------------------------------------------------------------
extern std::atomic<unsigned long long> g_launches;  // product kernels launched (lutgemm_launch_count)
int num_sms();
cudaError_t ensure_smem_attr(const void* kernel);  // dynamic-smem opt-in, once per (kernel, device)
const cudaLaunchAttribute* pdl_attr();              // programmatic stream serialization

// one product kernel launch: PDL attribute, p.smem_bytes of dynamic shared memory
template <typename K>
inline cudaError_t launch(K kernel, int grid, const KParams& p, cudaStream_t st, int threads = kThreads) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t err = ensure_smem_attr(reinterpret_cast<const void*>(kernel));
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = p.smem_bytes > 0 ? p.smem_bytes : kSmemBytesBase;
  cfg.stream = st;
  cfg.attrs = const_cast<cudaLaunchAttribute*>(pdl_attr());
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, p);
}

// fused mode: CTA c -> (slice or sub-slice c / J, row group c % J); (c + 0.5) / J in fp32 is exact
// enough to floor correctly for any grid of the fused mode (c < 2^16, J <= 256)
__device__ __forceinline__ void fused_slot(const KParams& p, int& s, int& fj) {
  const int c = (int)blockIdx.x;
  s = (int)(((float)c + 0.5f) * p.rcp_J);
  fj = c - s * p.fused_J;
}

// per-kernel-family launchers (dispatch on q and the scale format ZM)
cudaError_t launch_gemv(const KParams& p, int grid, cudaStream_t st);
cudaError_t launch_reduce(const KParams& p, cudaStream_t st);
cudaError_t launch_batched(const KParams& p, int grid, cudaStream_t st);
cudaError_t launch_reduce_batched(const KParams& p, cudaStream_t st);
void plan_batched(const Shape& sh, int sms, KParams& p);
cudaError_t launch_smallb(const KParams& p, int grid, cudaStream_t st);

// q -> compile-time QT (1..4, else 8 = up to 8 planes at runtime), ZM from the shape
template <template <int, int> class F>
inline cudaError_t dispatch_qz(const KParams& p, int grid, cudaStream_t st) {
  auto byq = [&](auto zm) -> cudaError_t {
    constexpr int ZM = decltype(zm)::value;
    switch (p.sh.q) {
      case 1: return F<1, ZM>::run(p, grid, st);
      case 2: return F<2, ZM>::run(p, grid, st);
      case 3: return F<3, ZM>::run(p, grid, st);
      case 4: return F<4, ZM>::run(p, grid, st);
      default: return F<8, ZM>::run(p, grid, st);
    }
  };
  if (p.sh.gcls == kGrpChunk) {  // per-chunk scales: the generic-q kernels only (ring_compute_cg)
    if (p.sh.has_z) return F<8, 1>::run(p, grid, st);
    return F<8, 0>::run(p, grid, st);
  }
  if (p.sh.compact) return byq(std::integral_constant<int, 2>{});
  if (p.sh.has_z) return byq(std::integral_constant<int, 1>{});
  return byq(std::integral_constant<int, 0>{});
}

}  // namespace lg
