// Packed e2m1 (FP4) copies of small-integer couplings for the kind::mxf4 tensor-core path.
//
// e2m1 = sign | 2-bit exponent (bias 1) | 1-bit mantissa; its exact integers are
// 0, 1, 2, 3, 4, 6 (codes 0x0, 0x2, 0x4, 0x5, 0x6, 0x7; negative: | 0x8). A J whose
// entries all lie in {0, +-1, +-2, +-3, +-4, +-6} (every +-1 instance: C1/C2/C5) is
// stored two entries per byte, the even column in the low nibble, [rows][kpad / 2].
#pragma once

#include <cstdint>

namespace sbg {

// e2m1 code of an int8 coupling, or 0xFF if it is not exactly representable.
__device__ __forceinline__ uint32_t e2m1_code(int v) {
  const int a = v < 0 ? -v : v;
  const uint32_t m = a == 0 ? 0u : a == 1 ? 2u : a == 2 ? 4u : a == 3 ? 5u : a == 4 ? 6u : a == 6 ? 7u : 0xFFu;
  return m == 0xFFu ? m : (m | (v < 0 ? 8u : 0u));
}

// J4[b] = code(J[2b]) | code(J[2b + 1]) << 4 over `bytes` output bytes (16 per thread
// per iteration); *bad is set if any entry is not e2m1-exact.
__global__ void pack_e2m1_kernel(const int8_t* __restrict__ J, uint8_t* __restrict__ J4, size_t bytes,
                                 unsigned* bad) {
  const size_t n16 = bytes / 16;
  unsigned b = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
    const int4 w0 = reinterpret_cast<const int4*>(J)[2 * i], w1 = reinterpret_cast<const int4*>(J)[2 * i + 1];
    const uint32_t in[8] = {uint32_t(w0.x), uint32_t(w0.y), uint32_t(w0.z), uint32_t(w0.w),
                            uint32_t(w1.x), uint32_t(w1.y), uint32_t(w1.z), uint32_t(w1.w)};
    uint32_t out[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t o = 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t word = in[2 * q + h];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t c = e2m1_code(static_cast<int8_t>(word >> (8 * e)));
          b |= c >> 4;
          o |= (c & 0xFu) << (4 * (4 * h + e));
        }
      }
      out[q] = o;
    }
    reinterpret_cast<uint4*>(J4)[i] = make_uint4(out[0], out[1], out[2], out[3]);
  }
  if (b) atomicOr(bad, 1u);
}

}  // namespace sbg
