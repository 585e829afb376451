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

// Two spins at once on the packed FP32 pipe (fma.rn.f32x2, sm_100). Every
// operation of gsb_phase is an FMA with an exact identity operand:
//   a*b = fma(a, b, -0)   a+b = fma(a, 1, b)   a-b = fma(b, -1, a)
// each equal to the correctly rounded scalar op (signed zeros included), so
// the pair update is bitwise gsb_phase applied to each lane. The identity
// operands MUST be runtime values (kernel arguments): with literal -0 / 1 / -1
// ptxas rewrites the FMAs into FMUL2 / FADD2 and then contracts those pairs
// back into FFMA2, changing the rounding.
namespace f2 {
__device__ __forceinline__ uint64_t pk(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
}  // namespace f2

struct PhaseIdent {  // -0, 1, -1 supplied at run time (see above)
  float mzero, one, mone;
};

struct PhaseConsts2 {
  uint64_t a, c, dt, inv, mzero, one, mone;
  __device__ __forceinline__ PhaseConsts2(const PhaseConsts& k, const PhaseIdent& id)
      : a(f2::pk(k.a, k.a)), c(f2::pk(k.c, k.c)), dt(f2::pk(k.dt, k.dt)), inv(f2::pk(k.inv, k.inv)),
        mzero(f2::pk(id.mzero, id.mzero)), one(f2::pk(id.one, id.one)), mone(f2::pk(id.mone, id.mone)) {}
};

// The strict walls of gsb_phase, branch-free: one |xn| > 1 test (false for NaN, like both
// of gsb_phase's tests), then +-1 = copysign(1, xn) by a bit operation, and y = +0.
__device__ __forceinline__ float clamp_wall(float xn, float& yn) {
  const bool out = fabsf(xn) > 1.0f;
  yn = out ? 0.0f : yn;
  return out ? __uint_as_float((__float_as_uint(xn) & 0x80000000u) | 0x3F800000u) : xn;
}

// (x0, x1), (y0, y1), (p0, p1) updated with fields F0, F1; a2 = packed A per lane.
__device__ __forceinline__ void gsb_phase2(float F0, float F1, float& x0, float& x1, float& y0, float& y1, float& p0,
                                           float& p1, const PhaseConsts2& k, uint64_t a2) {
  using namespace f2;
  const uint64_t x = pk(x0, x1), y = pk(y0, y1), p = pk(p0, p1), F = pk(F0, F1);
  const uint64_t ax2 = fma(fma(a2, x, k.mzero), x, k.mzero);
  const uint64_t g = fma(ax2, k.mone, k.one);
  const uint64_t pn = fma(fma(fma(g, p, k.mzero), k.inv, k.mzero), k.mone, p);
  const uint64_t t = fma(fma(k.c, F, k.mzero), k.mone, fma(pn, x, k.mzero));
  const uint64_t yn = fma(fma(t, k.dt, k.mzero), k.mone, y);
  const uint64_t xn = fma(fma(yn, k.dt, k.mzero), k.one, x);
  float xa, xb, ya, yb;
  upk(xn, xa, xb);
  upk(yn, ya, yb);
  upk(pn, p0, p1);
  x0 = clamp_wall(xa, ya);
  x1 = clamp_wall(xb, yb);
  y0 = ya;
  y1 = yb;
}

// q = rint(x * 2^30): the fixed-point image of x fed to the int8 tensor cores
// as four byte planes (signed base-256 digits, qdigits). |x| <= 1 so |q| <= 2^30.
__device__ __forceinline__ int32_t quant30(float x) { return __float2int_rn(__fmul_rn(x, 0x1p30f)); }

// q as four SIGNED base-256 digits d_p in [-128, 127], q = sum_p d_p 2^(8p), packed one
// per byte (plane p = byte p). Adding 128 to each of the three low bytes (with carries)
// and flipping their top bits back gives the balanced digits: d_p = u_p - 128 for p < 3
// and d_3 = u >> 24 (|q| <= 2^30 keeps it in [-64, 64]). Every plane is then s8, so one
// MMA instruction can take all planes of the B operand; the field sum_p 2^(8p) (J . d_p)
// is the same integer J . q as with unsigned low planes.
__device__ __forceinline__ uint32_t qdigits(int32_t q) {
  return static_cast<uint32_t>(q + 0x00808080) ^ 0x00808080u;
}

// sgn with sgn(0) = +1 (model.cpp:161-165, engine.cpp:73-77).
__device__ __forceinline__ int8_t sgn8(float x) { return x >= 0.0f ? int8_t(1) : int8_t(-1); }

}  // namespace sbg
