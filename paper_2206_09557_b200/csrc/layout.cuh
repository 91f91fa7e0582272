// layout.cuh -- the kernel-native HBM layout of a packed LUT-GEMM weight.
//
// Columns are cut into LUT slices of 1024 (= 128 mu=8 chunks = 128 tables of
// 256 fp32 = 128 KB of shared memory per CTA; App. B P:L589 "1KB ... for every
// 8 hidden dimensions").  Inside a slice, "layout lane" p owns the 32 columns
// [32p, 32p+32) = chunks 4p..4p+3, i.e. one canonical uint32 word per row.  The
// last slice of an n that is not a multiple of 1024 has fewer lanes (L < 32).
//
// The weight is ONE byte stream, slice-major; inside slice s it is a sequence
// of fixed-size records, one per row quad rq (rows 4rq..4rq+3):
//
//   record(s, rq) = keys  [q][L_s][4 rows] uint32   (q*L_s*16 bytes)
//                   alpha [gps_s][q][4 rows] fp16    (q*gps_s*8 bytes)
//                   z     [gps_s][4 rows] fp16       (gps_s*8 bytes, if has_offset)
//                   zero padding to a multiple of 16 bytes
//
// gps_s = groups per slice = 32*L_s/g when g <= 1024 (g must divide 1024), else
// 1 (g a multiple of 1024, or g == n): that group's scales are then repeated in
// every slice it spans.  So a CTA working on (slice s, row quads [a, b)) reads
// one contiguous byte range -- which a single bulk L2 prefetch can run ahead
// of -- and a warp's 128-bit key loads for one (rq, plane) cover 512
// contiguous bytes.  Rows m..m4-1 (m4 = 4*ceil(m/4)) are zero.
#pragma once
#include <cstddef>
#include <cstdint>

namespace lg {

constexpr int kSliceCols = 1024;
constexpr int kLanesPerSlice = 32;
constexpr int kLutBytes = 128 * 1024;

struct Shape {
  int m, n, q, g, has_z;
  int m4, RQ, G, S;
};

__host__ __device__ inline Shape make_shape(int m, int n, int q, int g, int has_z) {
  Shape s;
  s.m = m; s.n = n; s.q = q; s.g = g; s.has_z = has_z ? 1 : 0;
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

__host__ __device__ inline int slice_groups(const Shape& sh, int Ls) {
  return sh.g <= kSliceCols ? (32 * Ls) / sh.g : 1;
}

// group (within the slice's alpha block) of layout lane p
__host__ __device__ inline int lane_group(const Shape& sh, int p) {
  return sh.g <= kSliceCols ? (32 * p) / sh.g : 0;
}

// global group index of slice-local group k
__host__ __device__ inline int global_group(const Shape& sh, int s, int k) {
  return sh.g <= kSliceCols ? s * (kSliceCols / sh.g) + k : (s * kSliceCols) / sh.g;
}

__host__ __device__ inline uint32_t keys_bytes(const Shape& sh, int Ls) { return (uint32_t)sh.q * Ls * 16u; }

__host__ __device__ inline uint32_t record_bytes(const Shape& sh, int Ls) {
  const uint32_t gps = (uint32_t)slice_groups(sh, Ls);
  const uint32_t raw = keys_bytes(sh, Ls) + (uint32_t)sh.q * gps * 8u + (sh.has_z ? gps * 8u : 0u);
  return (raw + 15u) / 16u * 16u;
}

__host__ __device__ inline size_t slice_base(const Shape& sh, int s) {
  // every slice before s is full
  return (size_t)s * (size_t)sh.RQ * record_bytes(sh, kLanesPerSlice);
}

__host__ __device__ inline size_t record_offset(const Shape& sh, int s, int Ls, int rq) {
  return slice_base(sh, s) + (size_t)rq * record_bytes(sh, Ls);
}

__host__ __device__ inline size_t packed_bytes(const Shape& sh) {
  const int Sfull = sh.n / kSliceCols;
  size_t b = (size_t)Sfull * sh.RQ * record_bytes(sh, kLanesPerSlice);
  if (sh.n % kSliceCols) b += (size_t)sh.RQ * record_bytes(sh, slice_lanes(sh.n, Sfull));
  return b;
}

// byte offsets inside a record
__host__ __device__ inline uint32_t key_off(int Ls, int i, int p, int r4) {
  return ((uint32_t)i * Ls + p) * 16u + 4u * r4;
}
__host__ __device__ inline uint32_t alpha_off(const Shape& sh, int Ls, int i, int k, int r4) {
  return keys_bytes(sh, Ls) + ((uint32_t)k * sh.q + i) * 8u + 2u * r4;
}
__host__ __device__ inline uint32_t z_off(const Shape& sh, int Ls, int k, int r4) {
  return keys_bytes(sh, Ls) + (uint32_t)sh.q * slice_groups(sh, Ls) * 8u + k * 8u + 2u * r4;
}

}  // namespace lg
