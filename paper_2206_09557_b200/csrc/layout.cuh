// layout.cuh -- the kernel-native HBM layout of a packed LUT-GEMM weight.
//
// Columns are cut into LUT slices of 1024 (= 128 mu=8 chunks = 128 tables of
// 256 fp32 = 128 KB of shared memory per CTA, App. B P:L589 "1KB ... for every
// 8 hidden dimensions").  Inside a slice, "layout lane" p owns the 32 columns
// [32p, 32p+32) = chunks 4p..4p+3, i.e. one canonical uint32 word per row.  The
// last slice of an n that is not a multiple of 1024 has fewer lanes (L < 32).
//
// planes (bytes): slice-major; inside slice s (L_s lanes), for row quad rq
// (rows 4rq..4rq+3) and plane i, the L_s lanes' 16-byte vectors are contiguous:
//     off = base_s + ((rq*q + i)*L_s + p)*16 + r4*4     (one uint32 per row)
// with base_s = s * RQ*q*512 (all earlier slices are full).  A warp's LDG.128
// over the 32 lanes of one (rq, i) therefore reads 512 contiguous bytes.
//
// alpha (fp16): [RQ][q][G][4] -- the 4 rows of a quad are innermost, so a lane
// fetches (alpha of its group, plane i) for its 4 rows with one 8-byte load.
// offset z (fp16): [RQ][G][4].
// Rows m..m4-1 (m4 = 4*ceil(m/4)) are zero bits with zero scales.
#pragma once
#include <cstddef>
#include <cstdint>

namespace lg {

constexpr int kSliceCols = 1024;
constexpr int kLanesPerSlice = 32;
constexpr int kLutBytes = 128 * 1024;

struct Shape {
  int m, n, q, g;
  int m4, RQ, G, S;
};

__host__ __device__ inline Shape make_shape(int m, int n, int q, int g) {
  Shape s;
  s.m = m; s.n = n; s.q = q; s.g = g;
  s.m4 = (m + 3) / 4 * 4;
  s.RQ = s.m4 / 4;
  s.G = n / g;
  s.S = (n + kSliceCols - 1) / kSliceCols;
  return s;
}

__host__ __device__ inline int slice_lanes(int n, int s) {
  int rem = n - s * kSliceCols;
  return rem >= kSliceCols ? kLanesPerSlice : rem / 32;
}

__host__ __device__ inline size_t slice_base(const Shape& sh, int s) {
  return (size_t)s * (size_t)sh.RQ * (size_t)sh.q * 512u;
}

__host__ __device__ inline size_t plane_vec_offset(const Shape& sh, int s, int Ls, int rq, int i, int p) {
  return slice_base(sh, s) + (((size_t)rq * sh.q + i) * Ls + p) * 16u;
}

__host__ __device__ inline size_t planes_bytes(const Shape& sh) {
  return (size_t)sh.m4 * sh.q * (size_t)sh.n / 8u;
}
__host__ __device__ inline size_t alpha_elems(const Shape& sh) {
  return (size_t)sh.m4 * sh.G * sh.q;
}
__host__ __device__ inline size_t alpha_index(const Shape& sh, int rq, int i, int grp, int r4) {
  return (((size_t)rq * sh.q + i) * sh.G + grp) * 4u + r4;
}
__host__ __device__ inline size_t offset_elems(const Shape& sh) {
  return (size_t)sh.m4 * sh.G;
}
__host__ __device__ inline size_t offset_index(const Shape& sh, int rq, int grp, int r4) {
  return ((size_t)rq * sh.G + grp) * 4u + r4;
}

}  // namespace lg
