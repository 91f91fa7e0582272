// layout.cuh -- the kernel-native HBM layout of a packed LUT-GEMM weight.
//
// Columns are cut into LUT slices of 1024 (= 128 mu=8 chunks = 128 tables of
// 256 fp32 = 128 KB of shared memory per CTA; App. B P:L589 "1KB ... for every
// 8 hidden dimensions").  Inside a slice, "layout lane" p owns the 32 columns
// [32p, 32p+32) = chunks 4p..4p+3, i.e. one canonical uint32 word per row.  The
// last slice of an n that is not a multiple of 1024 has fewer lanes (L < 32).
//
// The weight is ONE buffer, slice-major.  Slice s holds three regions, each
// starting on a 256-byte boundary (the L2 fills DRAM sectors in 256-byte
// blocks; misaligned 512-byte warp loads would over-fetch):
//
//   keys  [RQ][q][L_s][4 rows] uint32   -> q*L_s*16 bytes per row quad
//   alpha [RQ][gps_s][qa][4 rows] fp16  -> qa*gps_s*8 bytes per row quad
//         (qa = q; compact uniform format: qa = 1, the stored value is s and
//         alpha_i = 2^(i-1) s is derived in the kernel, App. C)
//   z     [RQ][gps_s][4 rows] fp16      -> gps_s*8 bytes per row quad (has_offset)
//
// gps_s = scale groups stored per slice (slice_groups):
//   g == n (row-wise) or g a multiple of 1024: 1 -- the group's scales are
//     repeated in every slice it spans;
//   g | 1024 (g % 32 == 0): 32*L_s/g;
//   other g % 32 == 0 (e.g. 96, 384, 640, 1536): every group that intersects
//     the slice, a group straddling a slice boundary stored in both slices
//     (alpha (P1 + P2) = alpha P1 + alpha P2); a fixed bound (g + 991)/g + 1
//     per slice keeps the slice stride uniform (unused entries are zero);
//   g % 32 != 0 ("chunk groups", cg: g in {8, 16, 24, 40, ...}, P:L295-296
//     allows any g): one scale entry per 8-column chunk, 4 L_s per slice,
//     each holding its chunk's group scale; the alpha block of a row quad is
//     then [L_s lanes][qa][4 chunks][4 rows] so a lane's 4 chunks of one plane
//     are 32 contiguous bytes.
// n need only be a multiple of 8: the last lane of the last slice may be
// partial; its padding key bits are 0 and the kernels stage x as zero there.
// So a CTA working on (slice s, row quads [a, b)) reads three contiguous byte
// ranges, and a warp's 128-bit key loads for one (rq, plane) cover 512
// contiguous, 512-byte-aligned bytes (full slices).  Rows m..m4-1
// (m4 = 4*ceil(m/4)) are zero.
#pragma once
#include <cstddef>
#include <cstdint>

namespace lg {

constexpr int kSliceCols = 1024;
constexpr int kLanesPerSlice = 32;
constexpr int kLutBytes = 128 * 1024;

// group classes (see the header comment)
enum : int { kGrpOne = 0, kGrpDiv = 1, kGrpSpan = 2, kGrpChunk = 3 };

struct Shape {
  int m, n, q, g, has_z;
  int compact;  // 1: uniform-compact format (one stored scale s per group, has_z = 1)
  int gcls;     // group class: kGrpOne (row-wise / multiple of 1024), kGrpDiv (g | 1024), kGrpSpan, kGrpChunk
  int lsh;      // kGrpDiv: log2(g / 32), a layout lane's group is p >> lsh (g / 32 is a power of two)
  int m4, RQ, G, S;
};

__host__ __device__ inline int group_class(int n, int g) {
  if (g == n || (g >= kSliceCols && g % kSliceCols == 0)) return kGrpOne;
  if (g % 32) return kGrpChunk;
  if (g <= kSliceCols && kSliceCols % g == 0) return kGrpDiv;
  return kGrpSpan;
}

__host__ __device__ inline Shape make_shape(int m, int n, int q, int g, int has_z, int compact = 0) {
  Shape s;
  s.m = m; s.n = n; s.q = q; s.g = g; s.has_z = (has_z || compact) ? 1 : 0;
  s.compact = compact ? 1 : 0;
  s.gcls = group_class(n, g);
  s.lsh = 0;
  while (s.gcls == kGrpDiv && (32 << s.lsh) < g) ++s.lsh;
  s.m4 = (m + 3) / 4 * 4;
  s.RQ = s.m4 / 4;
  s.G = (n + g - 1) / g;
  s.S = (n + kSliceCols - 1) / kSliceCols;
  return s;
}

// layout lanes (32-column words) of slice s; the last one may be partial (n % 32 != 0)
__host__ __device__ inline int slice_lanes(int n, int s) {
  int rem = n - s * kSliceCols;
  return rem >= kSliceCols ? kLanesPerSlice : (rem + 31) / 32;
}

// valid columns of slice s
__host__ __device__ inline int slice_cols(int n, int s) {
  int rem = n - s * kSliceCols;
  return rem >= kSliceCols ? kSliceCols : rem;
}

// scale entries stored per (row, slice) of a slice with Ls lanes
__host__ __device__ inline int slice_groups(const Shape& sh, int Ls) {
  switch (sh.gcls) {
    case kGrpOne: return 1;
    case kGrpDiv: return (32 * Ls) / sh.g;
    case kGrpSpan: return (sh.g + kSliceCols - 33) / sh.g + 1;
    default: return 4 * Ls;
  }
}

// slice-local scale entry of layout lane p of slice s (kGrpChunk: of the lane's first chunk; its
// chunk j is entry 4p + j)
__host__ __device__ inline int lane_group(const Shape& sh, int s, int p) {
  switch (sh.gcls) {
    case kGrpOne: return 0;
    case kGrpDiv: return p >> sh.lsh;
    case kGrpSpan: return (s * kSliceCols + 32 * p) / sh.g - (s * kSliceCols) / sh.g;
    default: return 4 * p;
  }
}

// global group of slice-local scale entry k of slice s (may be >= G for unused kGrpSpan entries)
__host__ __device__ inline int global_group(const Shape& sh, int s, int k) {
  switch (sh.gcls) {
    case kGrpOne: return (int)(((long long)s * kSliceCols) / sh.g);
    case kGrpDiv: return s * (kSliceCols / sh.g) + k;
    case kGrpSpan: return (s * kSliceCols) / sh.g + k;
    default: return (s * kSliceCols + 8 * k) / sh.g;
  }
}

// first slice that stores group grp, and the group's entry there (its first chunk for kGrpChunk)
__host__ __device__ inline void home_of_group(const Shape& sh, int grp, int* s, int* k) {
  const long long c0 = (long long)grp * sh.g;  // the group's first column
  *s = (int)(c0 / kSliceCols);
  switch (sh.gcls) {
    case kGrpOne: *k = 0; break;
    case kGrpDiv: *k = grp % (kSliceCols / sh.g); break;
    case kGrpSpan: *k = grp - (*s * kSliceCols) / sh.g; break;
    default: *k = (int)((c0 - (long long)*s * kSliceCols) / 8);
  }
}

// bytes per row quad in each region
__host__ __device__ inline uint32_t keys_bytes(const Shape& sh, int Ls) { return (uint32_t)sh.q * Ls * 16u; }
// stored scales per (row, group): q alphas, or the single s of the compact format
__host__ __device__ inline int scale_planes(const Shape& sh) { return sh.compact ? 1 : sh.q; }
__host__ __device__ inline uint32_t alpha_bytes(const Shape& sh, int Ls) {
  return (uint32_t)scale_planes(sh) * slice_groups(sh, Ls) * 8u;
}
__host__ __device__ inline uint32_t z_bytes(const Shape& sh, int Ls) {
  return sh.has_z ? (uint32_t)slice_groups(sh, Ls) * 8u : 0u;
}

__host__ __device__ inline size_t pad256(size_t v) { return (v + 255) / 256 * 256; }

__host__ __device__ inline size_t slice_bytes(const Shape& sh, int Ls) {
  return pad256((size_t)sh.RQ * keys_bytes(sh, Ls)) + pad256((size_t)sh.RQ * alpha_bytes(sh, Ls)) +
         pad256((size_t)sh.RQ * z_bytes(sh, Ls));
}

__host__ __device__ inline size_t slice_base(const Shape& sh, int s) {
  return (size_t)s * slice_bytes(sh, kLanesPerSlice);  // every slice before s is full
}

// region bases inside the buffer
__host__ __device__ inline size_t keys_base(const Shape& sh, int s, int Ls) { return slice_base(sh, s); }
__host__ __device__ inline size_t alpha_base(const Shape& sh, int s, int Ls) {
  return slice_base(sh, s) + pad256((size_t)sh.RQ * keys_bytes(sh, Ls));
}
__host__ __device__ inline size_t z_base(const Shape& sh, int s, int Ls) {
  return alpha_base(sh, s, Ls) + pad256((size_t)sh.RQ * alpha_bytes(sh, Ls));
}

__host__ __device__ inline size_t packed_bytes(const Shape& sh) {
  const int Sfull = sh.n / kSliceCols;
  size_t b = (size_t)Sfull * slice_bytes(sh, kLanesPerSlice);
  if (sh.n % kSliceCols) b += slice_bytes(sh, slice_lanes(sh.n, Sfull));
  return b;
}

// byte offsets of single elements
__host__ __device__ inline size_t key_at(const Shape& sh, int s, int Ls, int rq, int i, int p, int r4) {
  return keys_base(sh, s, Ls) + (size_t)rq * keys_bytes(sh, Ls) + ((uint32_t)i * Ls + p) * 16u + 4u * r4;
}
__host__ __device__ inline size_t alpha_at(const Shape& sh, int s, int Ls, int rq, int i, int k, int r4) {
  const uint32_t qa = (uint32_t)scale_planes(sh);
  const uint32_t e = sh.gcls == kGrpChunk ? ((uint32_t)(k >> 2) * qa + i) * 4u + (k & 3) : (uint32_t)k * qa + i;
  return alpha_base(sh, s, Ls) + (size_t)rq * alpha_bytes(sh, Ls) + e * 8u + 2u * r4;
}
__host__ __device__ inline size_t z_at(const Shape& sh, int s, int Ls, int rq, int k, int r4) {
  return z_base(sh, s, Ls) + (size_t)rq * z_bytes(sh, Ls) + (uint32_t)k * 8u + 2u * r4;
}

}  // namespace lg
