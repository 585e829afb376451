// gen_random_dense (model.cpp:144-159) evaluated on the device, in the reference's
// exact draw order, for any n (C5's n = 100000 is 5e9 draws and 10 GB of int8 J,
// which the reference's serial fp64 generator cannot produce at all).
//
// The reference walks the strict upper triangle row-major and takes one
// Xoshiro256pp draw per pair (i < j): J_ij = J_ji = top bit of next() ? -1 : +1.
// Draw t of row i sits at stream index off(i) + (j - i - 1), with
// off(i) = i(n-1) - i(i-1)/2. The xoshiro256 state transition is linear over
// GF(2), so the state after d draws is T^d s0: the host squares the 256x256 bit
// matrix T into M_k = T^(2^k) once, and each device thread jumps straight to the
// start of its segment (<= 2048 pairs of one row) by applying M_k for the set bits
// of d, then runs the ordinary generator. Segments are independent, so the whole
// triangle is generated in parallel and bit-identical to the serial walk.
#pragma once

#include <cstdint>
#include <vector>

#include "aux_kernels.cuh"

namespace sbg {

constexpr int GEN_MAXK = 48;      // jump distances < 2^48 (n < 2^24.5)
constexpr int GEN_SEG = 2048;     // pairs per thread (multiple of 8)

// ---------------------------------------------------------------- host: T^(2^k)

inline void xo_transition(uint64_t s[4]) {  // rng.hpp next() without the output scrambler
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

// cols[k][b] = M_k e_b (4 words each), k < kmax.
inline std::vector<uint64_t> gen_jump_matrices(int kmax) {
  std::vector<uint64_t> cols(size_t(kmax) * 256 * 4, 0);
  for (int b = 0; b < 256; ++b) {
    uint64_t s[4] = {0, 0, 0, 0};
    s[b >> 6] = uint64_t(1) << (b & 63);
    xo_transition(s);
    for (int w = 0; w < 4; ++w) cols[size_t(b) * 4 + w] = s[w];
  }
  for (int k = 1; k < kmax; ++k) {
    const uint64_t* prev = &cols[size_t(k - 1) * 1024];
    uint64_t* cur = &cols[size_t(k) * 1024];
    for (int b = 0; b < 256; ++b) {  // M_k e_b = M_{k-1} (M_{k-1} e_b)
      const uint64_t* x = prev + size_t(b) * 4;
      uint64_t o[4] = {0, 0, 0, 0};
      for (int c = 0; c < 256; ++c)
        if ((x[c >> 6] >> (c & 63)) & 1)
          for (int w = 0; w < 4; ++w) o[w] ^= prev[size_t(c) * 4 + w];
      for (int w = 0; w < 4; ++w) cur[size_t(b) * 4 + w] = o[w];
    }
  }
  return cols;
}

// --------------------------------------------------------------------- device

__device__ __forceinline__ uint64_t gen_pair_offset(int64_t n, int64_t i) {  // off(i)
  return uint64_t(i) * uint64_t(n - 1) - uint64_t(i) * uint64_t(i - 1) / 2;
}

// s <- T^d s. Every thread of the warp walks the same k (uniform loads of the
// column table, broadcast); bits not set in d leave the state unchanged.
__device__ __forceinline__ void gen_jump(const ulonglong4* __restrict__ cols, int kmax, uint64_t d, uint64_t s[4]) {
  for (int k = 0; k < kmax; ++k) {
    const bool take = (d >> k) & 1;
    if (!__any_sync(0xffffffffu, take)) continue;
    const ulonglong4* mk = cols + size_t(k) * 256;
    uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint64_t x = s[w];
#pragma unroll 8
      for (int b = 0; b < 64; ++b) {
        const ulonglong2* c = reinterpret_cast<const ulonglong2*>(mk + w * 64 + b);
        const ulonglong2 lo = __ldg(c), hi = __ldg(c + 1);
        const uint64_t m = 0ull - ((x >> b) & 1ull);
        o0 ^= lo.x & m;
        o1 ^= lo.y & m;
        o2 ^= hi.x & m;
        o3 ^= hi.y & m;
      }
    }
    if (take) {
      s[0] = o0;
      s[1] = o1;
      s[2] = o2;
      s[3] = o3;
    }
  }
}

__device__ __forceinline__ int8_t gen_sign(Xoshiro& g) { return (g.next() >> 63) ? int8_t(-1) : int8_t(1); }

// Upper triangle, rows [r0, r1): out[(i - r0) * ld + j] for i < j < n, as whole
// aligned 8-byte words (bytes outside (i, n) written as 0; the lower triangle is
// filled afterwards). Thread = (row i, column segment s of GEN_SEG columns).
__global__ void gen_dense_upper_kernel(int8_t* __restrict__ out, int64_t ld, int64_t n, int64_t r0, int64_t r1,
                                       const ulonglong4* __restrict__ cols, int kmax, uint64_t seed, int seg) {
  const int64_t nseg = (n + seg - 1) / seg;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t i = r0 + t / nseg;
  const int64_t s = t % nseg;
  const bool live = i < r1 && i < n;
  const int64_t jb = live ? (i + 1 > s * seg ? i + 1 : s * seg) : n;
  const int64_t je = live ? (n < (s + 1) * int64_t(seg) ? n : (s + 1) * int64_t(seg)) : n;
  Xoshiro g(seed);
  uint64_t st[4] = {g.s0, g.s1, g.s2, g.s3};
  const uint64_t d = jb < je ? gen_pair_offset(n, i) + uint64_t(jb - i - 1) : 0;
  gen_jump(cols, kmax, d, st);
  if (jb >= je) return;
  g.s0 = st[0];
  g.s1 = st[1];
  g.s2 = st[2];
  g.s3 = st[3];
  int8_t* row = out + (i - r0) * ld;
  for (int64_t w0 = jb & ~int64_t(7); w0 < je; w0 += 8) {
    uint64_t word = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int64_t j = w0 + b;
      if (j >= jb && j < je) word |= uint64_t(uint8_t(gen_sign(g))) << (8 * b);
    }
    *reinterpret_cast<uint64_t*>(row + w0) = word;
  }
}

// Row-sharded lower part: rows [r0, r1) need J_ij = J_ji for j < i, i.e. the
// upper-triangle pairs (j, i) with i in [r0, r1). Thread = (row j, segment of the
// column window); byte scatter into out[(i - r0) * ld + j].
__global__ void gen_dense_strip_kernel(int8_t* __restrict__ out, int64_t ld, int64_t n, int64_t r0, int64_t r1,
                                       const ulonglong4* __restrict__ cols, int kmax, uint64_t seed, int seg) {
  const int64_t c1 = r1 < n ? r1 : n;
  const int64_t nseg = (c1 - r0 + seg - 1) / seg;
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t j = t / nseg;
  const int64_t s = t % nseg;
  const bool live = j < c1;
  const int64_t ib = live ? (j + 1 > r0 + s * seg ? j + 1 : r0 + s * seg) : c1;
  const int64_t ie = live ? (c1 < r0 + (s + 1) * int64_t(seg) ? c1 : r0 + (s + 1) * int64_t(seg)) : c1;
  Xoshiro g(seed);
  uint64_t st[4] = {g.s0, g.s1, g.s2, g.s3};
  const uint64_t d = ib < ie ? gen_pair_offset(n, j) + uint64_t(ib - j - 1) : 0;
  gen_jump(cols, kmax, d, st);
  if (ib >= ie) return;
  g.s0 = st[0];
  g.s1 = st[1];
  g.s2 = st[2];
  g.s3 = st[3];
  for (int64_t i = ib; i < ie; ++i) out[(i - r0) * ld + j] = gen_sign(g);
}

// Lower triangle of a square matrix from its upper triangle: J_ij = J_ji, i > j.
// 64x64 tiles through shared memory; CTA (bx, by) owns destination tile rows
// by*64.., columns bx*64.. with bx <= by.
__global__ void __launch_bounds__(256) mirror_lower_kernel(int8_t* __restrict__ J, int64_t ld, int64_t n) {
  const int64_t bx = blockIdx.x, by = blockIdx.y;
  if (bx > by) return;
  __shared__ __align__(16) uint8_t tile[64][64 + 16];
  const int tr = threadIdx.x >> 2, tc = (threadIdx.x & 3) * 16;
  // source: rows bx*64 + tr, columns by*64 + tc .. +16 (upper triangle side)
  const int64_t si = bx * 64 + tr, sj = by * 64 + tc;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (si < n && sj < ld) v = *reinterpret_cast<const uint4*>(J + si * ld + sj);
  *reinterpret_cast<uint4*>(&tile[tr][tc]) = v;
  __syncthreads();
  const int64_t di = by * 64 + tr;
  if (di >= n) return;
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 16; ++k) w[k >> 2] |= uint32_t(tile[tc + k][tr]) << (8 * (k & 3));
  int8_t* dst = J + di * ld + bx * 64 + tc;
  if (bx < by) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (bx * 64 + tc + k < di) dst[k] = int8_t(uint8_t(w[k >> 2] >> (8 * (k & 3))));
  }
}

}  // namespace sbg
