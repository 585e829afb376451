// The per-spin GSB phase update, fp32, in one fixed op order.
//
// Semantics: sbopt::step, /root/reference/proj/core/src/engine.cpp:86-103
//   p <- p - (1 - a x^2) p / (M - m)          (Eq. 7; a = 0 for bsb/dsb, :64)
//        computed as p - ((1 - a x^2) p) * inv, inv = RN(1 / (M - m)) (one
//        correctly rounded reciprocal per step instead of a per-spin divide)
//   y <- y - (p x - c F) dt
//   x <- x + y dt
//   |x| > 1  ->  x = sgn(x), y = 0            (strict walls, :93-99)
// with x read at t_m throughout. Every operation is an explicit round-to-
// nearest intrinsic (no FMA contraction), so the C mirror in
// oracle/sbg_oracle.c:orc_phase_f32 (compiled -ffp-contract=off) reproduces it
// bit for bit.
#pragma once

#include <cstdint>

namespace sbg {

struct PhaseConsts {
  float a;      // nonlinear control strength A (0 for bsb/dsb)
  float c;      // coupling scale
  float dt;     // time step
  float inv;    // RN(1 / (float)(M - m))
};

__device__ __forceinline__ void gsb_phase(float F, float& x, float& y, float& p, const PhaseConsts& k) {
  const float ax2 = __fmul_rn(__fmul_rn(k.a, x), x);
  const float g = __fsub_rn(1.0f, ax2);
  const float pn = __fsub_rn(p, __fmul_rn(__fmul_rn(g, p), k.inv));
  const float t = __fsub_rn(__fmul_rn(pn, x), __fmul_rn(k.c, F));
  float yn = __fsub_rn(y, __fmul_rn(t, k.dt));
  float xn = __fadd_rn(x, __fmul_rn(yn, k.dt));
  if (xn > 1.0f) {
    xn = 1.0f;
    yn = 0.0f;
  } else if (xn < -1.0f) {
    xn = -1.0f;
    yn = 0.0f;
  }
  x = xn;
  y = yn;
  p = pn;
}

// q = rint(x * 2^30): the fixed-point image of x fed to the int8 tensor cores
// as four byte planes (u8, u8, u8, s8). |x| <= 1 so |q| <= 2^30.
__device__ __forceinline__ int32_t quant30(float x) { return __float2int_rn(__fmul_rn(x, 0x1p30f)); }

// sgn with sgn(0) = +1 (model.cpp:161-165, engine.cpp:73-77).
__device__ __forceinline__ int8_t sgn8(float x) { return x >= 0.0f ? int8_t(1) : int8_t(-1); }

}  // namespace sbg
