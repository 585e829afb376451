// GSB step for sparse integer couplings (CSR, both triangles, int8 values).
//
// Same semantics as the dense step (engine.cpp:55-110 on the dense view of the
// instance); the field is the exact integer sum
//   sign variants:  F_i = sum_k val_k * sgn(x_{col_k})
//   fixed-point:    F_i = fl32(sum_k val_k * q_{col_k}) * 2^-30,  q = rint(x 2^30)
// which equals the dense tensor-core field bit for bit (zeros contribute 0).
//
// Layout: while stepping, the state lives SPIN-MAJOR ([npad][rp], replicas
// contiguous) so that the SpMM gather of row j for a block of replicas is one
// contiguous, vectorised read: a warp owns (row i, 128 CSR_VEC replicas), lane l holds
// replicas 4l..4l+3 (+ 128 u for CSR_VEC > 1; int4 / char4 / float4 accesses, one 512 B
// gather per warp per nonzero and group). CSR_VEC = 1 at 32 registers (8 blocks of 256
// threads per SM) measured 77.9 us/step at C3 vs 80.2 for CSR_VEC = 2 at 48 registers;
// with the gather address one IMAD.WIDE.U32 and no per-replica predicate, the nonzero loop
// not unrolled (no spills at 32 registers) gives 71.2 (unroll 2: 74.7, 4: 78.9; 48 warps
// with unroll 4: 91.7; an L2 prefetch of x, y, p at task start: 72.5);
// a variant that prefetches x, y, p and batches 4-8 gathers before use was slower
// (85-167 us: the extra registers cost more occupancy than the batching gains).
// The row's (col, val) pairs are loaded once, one per lane, and broadcast with
// shuffles, so all gathers of a row are independent (memory-level parallelism).
// The gathered operand (q or sgn x) is ping-ponged between two buffers because
// other warps still read step t's values while row i writes step t+1's;
// x, y, p are owned by row i and updated in place. The sbgpu API keeps the
// replica-major layout; sbg_advance transposes in and out once per call.
#pragma once

#include <cstdint>
#include <type_traits>

#include "gsb_phase.cuh"

namespace sbg {

constexpr int CSR_THREADS = 256;
// the gathers of the ping-pong operand: random 512 B rows with no reuse inside an SM
#ifndef CSR_GATHER_LD
#define CSR_GATHER_LD "ld.global.L2::cache_hint"  // L1::no_allocate measured the same (68.5 us)
#endif
constexpr int CSR_VEC = 1;                     // 4-replica groups per lane (more gathers in flight)
constexpr int CSR_RCHUNK = 128 * CSR_VEC;      // replicas per warp task
#ifndef CSR_MINB
#define CSR_MINB 8
#endif
#ifndef CSR_UNROLL
#define CSR_UNROLL 1
#endif

#ifndef CSR_LEAN_DEFAULT
#define CSR_LEAN_DEFAULT 2  // gathers per round of csr_step_lean_kernel (SBG_CSR_LEAN overrides)
#endif
constexpr int CSR_UNR = CSR_UNROLL;             // nonzeros per unrolled gather round
constexpr int CSR_MIN_BLOCKS = CSR_MINB;       // 64 warps per SM: latency hiding for the gathers

// L2 eviction priorities: the x/y/p stream is touched once per step (evict_first);
// the gathered operand (q or signs, re-read ~degree times per step) should stay.
namespace l2 {
__device__ __forceinline__ uint64_t evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// the x, y, p stream: evict_first (one pass) by default; with replica slabs (state + operands
// sized to stay in L2 across the slab's steps) CSR_STATE_POLICY = 1 / 2 keeps it normal / last --
// measured slower at C3: 71.8 / 75.5 vs 69.6 us/step (and with 128-replica slabs 75.3 / 76.3 vs 80.7)
#ifndef CSR_STATE_POLICY
#define CSR_STATE_POLICY 0
#endif
__device__ __forceinline__ uint64_t state_policy() {
#if CSR_STATE_POLICY == 1
  return evict_normal();
#elif CSR_STATE_POLICY == 2
  return evict_last();
#else
  return evict_first();
#endif
}
__device__ __forceinline__ float4 ld_f4(const float* a, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_f4(float* a, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ int4 ld_i4(const int32_t* a, uint64_t pol) {
  int4 v;
  asm volatile(CSR_GATHER_LD ".v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_i4(int32_t* a, int4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint32_t ld_u32(const void* a, uint64_t pol) {
  uint32_t v;
  asm volatile(CSR_GATHER_LD ".u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_u32(void* a, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}
}  // namespace l2

template <bool SIGN>
__global__ void __launch_bounds__(CSR_THREADS, CSR_MIN_BLOCKS)
    csr_step_sm_kernel(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const int8_t* __restrict__ val, const void* __restrict__ g_cur, void* __restrict__ g_next,
                       float* __restrict__ xs, float* __restrict__ ys, float* __restrict__ ps, int64_t rp,
                       int32_t R, PhaseConsts k, const float* __restrict__ a_rep = nullptr) {
  const int lane = threadIdx.x & 31;
  const int chunks = static_cast<int>((R + CSR_RCHUNK - 1) / CSR_RCHUNK);
  const int64_t tasks = static_cast<int64_t>(n) * chunks;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t stream = l2::state_policy(), keep = l2::evict_last();
  // row stride of the gathered operand in bytes: row j of a lane's group is one IMAD.WIDE.U32 away
  const uint32_t rsb = static_cast<uint32_t>(rp) * (SIGN ? 1u : 4u);
  for (int64_t t = wid; t < tasks; t += nw) {
    const int i = static_cast<int>(t / chunks);
    const int rc = static_cast<int>(t % chunks) * CSR_RCHUNK + 4 * lane;  // group u covers rc + 128 u .. +3
    const int kb = rowptr[i], ke = rowptr[i + 1];
    // every lane gathers, padding replicas (rc >= R, inside rp) included: no predicate in the loop
    const char* gb[CSR_VEC];
#pragma unroll
    for (int u = 0; u < CSR_VEC; ++u)
      gb[u] = static_cast<const char*>(g_cur) + static_cast<size_t>(rc + 128 * u) * (SIGN ? 1 : 4);
    long long acc[CSR_VEC][4];
#pragma unroll
    for (int u = 0; u < CSR_VEC; ++u) acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0;
    for (int k0 = kb; k0 < ke; k0 += 32) {
      const int cnt = min(32, ke - k0);
      int jl = 0, vl = 0;
      if (lane < cnt) {
        jl = col[k0 + lane];
        vl = val[k0 + lane];
      }
#pragma unroll CSR_UNR
      for (int kk = 0; kk < cnt; ++kk) {
        const int j = __shfl_sync(0xffffffffu, jl, kk);
        const long long v = __shfl_sync(0xffffffffu, vl, kk);
#pragma unroll
        for (int u = 0; u < CSR_VEC; ++u) {
          const char* src = gb[u] + static_cast<uint64_t>(static_cast<uint32_t>(j)) * rsb;
          if (SIGN) {
            const uint32_t w = l2::ld_u32(src, keep);
            const char4 s = *reinterpret_cast<const char4*>(&w);
            acc[u][0] += v * s.x;
            acc[u][1] += v * s.y;
            acc[u][2] += v * s.z;
            acc[u][3] += v * s.w;
          } else {
            const int4 q = l2::ld_i4(reinterpret_cast<const int32_t*>(src), keep);
            acc[u][0] += v * q.x;
            acc[u][1] += v * q.y;
            acc[u][2] += v * q.z;
            acc[u][3] += v * q.w;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CSR_VEC; ++u) {
      const int r = rc + 128 * u;
      if (r >= R) continue;
      const size_t off = static_cast<size_t>(i) * rp + r;
      float4 x4 = l2::ld_f4(xs + off, stream);
      float4 y4 = l2::ld_f4(ys + off, stream);
      float4 p4 = l2::ld_f4(ps + off, stream);
      float F[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        F[e] = SIGN ? static_cast<float>(acc[u][e]) : __fmul_rn(__ll2float_rn(acc[u][e]), 0x1p-30f);
      PhaseConsts kk[4] = {k, k, k, k};
      if (a_rep) {
#pragma unroll
        for (int e = 0; e < 4; ++e) kk[e].a = a_rep[min(r + e, R - 1)];
      }
      gsb_phase(F[0], x4.x, y4.x, p4.x, kk[0]);
      gsb_phase(F[1], x4.y, y4.y, p4.y, kk[1]);
      gsb_phase(F[2], x4.z, y4.z, p4.z, kk[2]);
      gsb_phase(F[3], x4.w, y4.w, p4.w, kk[3]);
      // replicas >= R inside the last group are padding: their slots exist (rp) and stay inert
      l2::st_f4(xs + off, x4, stream);
      l2::st_f4(ys + off, y4, stream);
      l2::st_f4(ps + off, p4, stream);
      if (SIGN) {
        char4 s;
        s.x = sgn8(x4.x);
        s.y = sgn8(x4.y);
        s.z = sgn8(x4.z);
        s.w = sgn8(x4.w);
        l2::st_u32(static_cast<int8_t*>(g_next) + off, *reinterpret_cast<uint32_t*>(&s), keep);
      } else {
        l2::st_i4(static_cast<int32_t*>(g_next) + off,
                  make_int4(quant30(x4.x), quant30(x4.y), quant30(x4.z), quant30(x4.w)), keep);
      }
    }
  }
}

// The same step with fewer issued instructions per task (the step above runs at ~0.6 warp
// instructions per scheduler-cycle with 64 warps per SM: issue slots, not bytes, pace it).
//   * (row, chunk) advance incrementally per warp: no 64-bit division per task;
//   * the row's nonzeros are staged once per task in shared memory as (column, value) and read
//     back UNR at a time with one broadcast LDS.128 (the loop above spends two shuffles, their
//     convergence check, a constant reload and a 64-bit add per nonzero);
//   * the gather address is a 32-bit element index (column x rp + replica) and one scaled add;
//   * UNR nonzeros per round with their gathers issued back to back; a ragged tail gathers row 0
//     with value 0 (lanes >= cnt stage zeros), so the loop has no remainder code;
//   * the phase update runs two replicas at a time on the packed FP32 pipe (gsb_phase2, bitwise
//     gsb_phase), and all state addresses are 32-bit element offsets (host-checked: n * rp * 4 B
//     < 4 GB, else the kernel above runs).
// Same integer field, same update: bitwise equal (test_csr_kernel_variants_bitwise).
// PFS: the task's x, y, p (3 x 512 B per warp) are fetched into shared memory by cp.async at task
// start and read back after the gather loop, so their DRAM latency runs under the gathers instead
// of after them (ncu: 17 % of the stall samples sat on the first FFMA2 of the phase update) --
// without holding 12 registers across the loop.
template <bool SIGN, int UNR, bool PFS = false>
__global__ void __launch_bounds__(CSR_THREADS, CSR_MIN_BLOCKS)
    csr_step_lean_kernel(uint32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                         const int8_t* __restrict__ val, const void* __restrict__ g_cur, void* __restrict__ g_next,
                         float* __restrict__ xs, float* __restrict__ ys, float* __restrict__ ps, uint32_t rp,
                         uint32_t R, PhaseConsts k, PhaseIdent id, const float* __restrict__ a_rep = nullptr) {
  static_assert(UNR == 1 || UNR == 2 || UNR == 4, "gathers per round");
  __shared__ __align__(16) uint2 stage[CSR_THREADS / 32][32];  // (column, value) of the row's nonzeros
  __shared__ __align__(16) float4 sstate[PFS ? CSR_THREADS / 32 : 1][3][PFS ? 32 : 1];  // PFS: x, y, p of the task
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t chunks = (R + CSR_RCHUNK - 1) / CSR_RCHUNK;
  const uint32_t nw = gridDim.x * (CSR_THREADS / 32);
  const uint32_t di = nw / chunks, dc = nw - di * chunks;
  const uint32_t wid = blockIdx.x * (CSR_THREADS / 32) + wib;
  uint32_t i = wid / chunks, c = wid - i * chunks;
  const uint64_t stream = l2::state_policy(), keep = l2::evict_last();
  const uint32_t sp = static_cast<uint32_t>(__cvta_generic_to_shared(stage[wib]));  // this warp's 256 B
  const PhaseConsts2 k2(k, id);
  using Acc = std::conditional_t<SIGN, int32_t, long long>;
  while (i < n) {
    const uint32_t r = c * CSR_RCHUNK + 4 * lane;
    const int kb = rowptr[i], ke = rowptr[i + 1];
    Acc acc[4] = {0, 0, 0, 0};
    uint32_t ss = 0;
    if constexpr (PFS) {
      ss = static_cast<uint32_t>(__cvta_generic_to_shared(&sstate[wib][0][lane]));
      if (r < R) {
        const uint32_t off = i * rp + r;
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(ss), "l"(xs + off), "l"(stream)
                     : "memory");
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(ss + 512), "l"(ys + off),
                     "l"(stream)
                     : "memory");
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(ss + 1024), "l"(ps + off),
                     "l"(stream)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int k0 = kb; k0 < ke; k0 += 32) {
      const int cnt = min(32, ke - k0);
      uint32_t ej = 0, ev = 0;  // lanes >= cnt stage (row 0, value 0): the ragged tail of a round
      if (static_cast<int>(lane) < cnt) {
        ej = static_cast<uint32_t>(col[k0 + lane]);
        ev = static_cast<uint32_t>(static_cast<int32_t>(val[k0 + lane]));
      }
      __syncwarp();  // the previous round's reads are done
      asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(sp + lane * 8), "r"(ej), "r"(ev) : "memory");
      __syncwarp();
#pragma unroll 1
      for (uint32_t a = sp, ae = sp + static_cast<uint32_t>(cnt) * 8; a < ae; a += 8 * UNR) {
        uint32_t ew[2 * UNR];  // {col, val} x UNR, one broadcast load
        if constexpr (UNR == 1) {
          asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(ew[0]), "=r"(ew[1]) : "r"(a));
        } else {
#pragma unroll
          for (int h = 0; h < UNR / 2; ++h)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(ew[4 * h]), "=r"(ew[4 * h + 1]), "=r"(ew[4 * h + 2]), "=r"(ew[4 * h + 3])
                         : "r"(a + 16 * h));
        }
        // element index of the lane's group in row col (32-bit: host-checked), then one scaled add
        uint32_t src[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) src[u] = ew[2 * u] * rp + r;
        if constexpr (SIGN) {
          uint32_t w[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) w[u] = l2::ld_u32(static_cast<const int8_t*>(g_cur) + src[u], keep);
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            const int32_t v = static_cast<int32_t>(ew[2 * u + 1]);
            const char4 s = *reinterpret_cast<const char4*>(&w[u]);
            acc[0] += v * s.x;
            acc[1] += v * s.y;
            acc[2] += v * s.z;
            acc[3] += v * s.w;
          }
        } else {
          int4 q[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) q[u] = l2::ld_i4(static_cast<const int32_t*>(g_cur) + src[u], keep);
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            const long long v = static_cast<int32_t>(ew[2 * u + 1]);
            acc[0] += v * q[u].x;
            acc[1] += v * q[u].y;
            acc[2] += v * q[u].z;
            acc[3] += v * q[u].w;
          }
        }
      }
    }
    if constexpr (PFS) asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (r < R) {
      const uint32_t off = i * rp + r;
      float4 x4, y4, p4;
      if constexpr (PFS) {
        auto lds4 = [](uint32_t a) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
          return v;
        };
        x4 = lds4(ss);
        y4 = lds4(ss + 512);
        p4 = lds4(ss + 1024);
      } else {
        x4 = l2::ld_f4(xs + off, stream);
        y4 = l2::ld_f4(ys + off, stream);
        p4 = l2::ld_f4(ps + off, stream);
      }
      float F[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        F[e] = SIGN ? static_cast<float>(acc[e]) : __fmul_rn(__ll2float_rn(acc[e]), 0x1p-30f);
      uint64_t a01 = k2.a, a23 = k2.a;
      if (a_rep) {
        const uint32_t last = R - 1;
        a01 = f2::pk(a_rep[min(r, last)], a_rep[min(r + 1, last)]);
        a23 = f2::pk(a_rep[min(r + 2, last)], a_rep[min(r + 3, last)]);
      }
      gsb_phase2(F[0], F[1], x4.x, x4.y, y4.x, y4.y, p4.x, p4.y, k2, a01);
      gsb_phase2(F[2], F[3], x4.z, x4.w, y4.z, y4.w, p4.z, p4.w, k2, a23);
      // replicas >= R inside the last group are padding: their slots exist (rp) and stay inert
      l2::st_f4(xs + off, x4, stream);
      l2::st_f4(ys + off, y4, stream);
      l2::st_f4(ps + off, p4, stream);
      if (SIGN) {
        char4 s;
        s.x = sgn8(x4.x);
        s.y = sgn8(x4.y);
        s.z = sgn8(x4.z);
        s.w = sgn8(x4.w);
        l2::st_u32(static_cast<int8_t*>(g_next) + off, *reinterpret_cast<uint32_t*>(&s), keep);
      } else {
        l2::st_i4(static_cast<int32_t*>(g_next) + off,
                  make_int4(quant30(x4.x), quant30(x4.y), quant30(x4.z), quant30(x4.w)), keep);
      }
    }
    i += di;
    c += dc;
    if (c >= chunks) {
      c -= chunks;
      ++i;
    }
  }
}

// The register-path step with the gather loop software-pipelined by one: the load of nonzero
// k + 1 is issued before the accumulate of nonzero k, so every warp keeps two gathers in
// flight (the plain loop issues the next load only after the previous one's accumulate has
// waited for it). Four more registers per thread; MINB blocks of 256 threads per SM. Dev
// variant (SBG_CSR_PF=6/7), bitwise equal, measured slower at C3: 84.3 (6 blocks, 40 regs) /
// 91.7 (7 blocks, 32 regs + spills) vs 68.1 us/step -- like every other way of putting more
// gathers in flight (unroll, cp.async batches).
template <bool SIGN, int MINB>
__global__ void __launch_bounds__(CSR_THREADS, MINB)
    csr_step_pf_kernel(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const int8_t* __restrict__ val, const void* __restrict__ g_cur, void* __restrict__ g_next,
                       float* __restrict__ xs, float* __restrict__ ys, float* __restrict__ ps, int64_t rp,
                       int32_t R, PhaseConsts k, const float* __restrict__ a_rep = nullptr) {
  const int lane = threadIdx.x & 31;
  const int chunks = static_cast<int>((R + CSR_RCHUNK - 1) / CSR_RCHUNK);
  const int64_t tasks = static_cast<int64_t>(n) * chunks;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t stream = l2::state_policy(), keep = l2::evict_last();
  const uint32_t rsb = static_cast<uint32_t>(rp) * (SIGN ? 1u : 4u);
  using G = std::conditional_t<SIGN, uint32_t, int4>;
  auto gather = [&](const char* src) -> G {
    if constexpr (SIGN)
      return l2::ld_u32(src, keep);
    else
      return l2::ld_i4(reinterpret_cast<const int32_t*>(src), keep);
  };
  for (int64_t t = wid; t < tasks; t += nw) {
    const int i = static_cast<int>(t / chunks);
    const int rc = static_cast<int>(t % chunks) * CSR_RCHUNK + 4 * lane;
    const int kb = rowptr[i], ke = rowptr[i + 1];
    const char* gb = static_cast<const char*>(g_cur) + static_cast<size_t>(rc) * (SIGN ? 1 : 4);
    long long acc[4] = {0, 0, 0, 0};
    for (int k0 = kb; k0 < ke; k0 += 32) {
      const int cnt = min(32, ke - k0);
      int jl = 0, vl = 0;
      if (lane < cnt) {
        jl = col[k0 + lane];
        vl = val[k0 + lane];
      }
      G nxt = gather(gb + static_cast<uint64_t>(static_cast<uint32_t>(__shfl_sync(0xffffffffu, jl, 0))) * rsb);
#pragma unroll 1
      for (int kk = 0; kk < cnt; ++kk) {
        const G cur = nxt;
        const int jn = __shfl_sync(0xffffffffu, jl, kk + 1 < cnt ? kk + 1 : kk);
        if (kk + 1 < cnt) nxt = gather(gb + static_cast<uint64_t>(static_cast<uint32_t>(jn)) * rsb);
        const long long v = __shfl_sync(0xffffffffu, vl, kk);
        if constexpr (SIGN) {
          const char4 sg = *reinterpret_cast<const char4*>(&cur);
          acc[0] += v * sg.x;
          acc[1] += v * sg.y;
          acc[2] += v * sg.z;
          acc[3] += v * sg.w;
        } else {
          acc[0] += v * cur.x;
          acc[1] += v * cur.y;
          acc[2] += v * cur.z;
          acc[3] += v * cur.w;
        }
      }
    }
    const int r = rc;
    if (r >= R) continue;
    const size_t off = static_cast<size_t>(i) * rp + r;
    float4 x4 = l2::ld_f4(xs + off, stream);
    float4 y4 = l2::ld_f4(ys + off, stream);
    float4 p4 = l2::ld_f4(ps + off, stream);
    float F[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      F[e] = SIGN ? static_cast<float>(acc[e]) : __fmul_rn(__ll2float_rn(acc[e]), 0x1p-30f);
    PhaseConsts kk4[4] = {k, k, k, k};
    if (a_rep) {
#pragma unroll
      for (int e = 0; e < 4; ++e) kk4[e].a = a_rep[min(r + e, R - 1)];
    }
    gsb_phase(F[0], x4.x, y4.x, p4.x, kk4[0]);
    gsb_phase(F[1], x4.y, y4.y, p4.y, kk4[1]);
    gsb_phase(F[2], x4.z, y4.z, p4.z, kk4[2]);
    gsb_phase(F[3], x4.w, y4.w, p4.w, kk4[3]);
    l2::st_f4(xs + off, x4, stream);
    l2::st_f4(ys + off, y4, stream);
    l2::st_f4(ps + off, p4, stream);
    if (SIGN) {
      char4 sg;
      sg.x = sgn8(x4.x);
      sg.y = sgn8(x4.y);
      sg.z = sgn8(x4.z);
      sg.w = sgn8(x4.w);
      l2::st_u32(static_cast<int8_t*>(g_next) + off, *reinterpret_cast<uint32_t*>(&sg), keep);
    } else {
      l2::st_i4(static_cast<int32_t*>(g_next) + off,
                make_int4(quant30(x4.x), quant30(x4.y), quant30(x4.z), quant30(x4.w)), keep);
    }
  }
}

// Same step with the gathers staged through shared memory by cp.async (register-free loads):
// a warp issues up to NB gathers of its row (and its x, y, p) before waiting once, so each
// warp keeps NB loads in flight where the register-path kernel keeps one (its accumulate
// consumes each gather before the next is issued, at 32 registers). Per warp: NB slots of
// 32 * EB bytes (EB = 16 for q, 4 for sign bytes) + 1.5 KB of x, y, p. Bitwise the same
// field and update as csr_step_sm_kernel (identical integer sums, same gsb_phase).
constexpr int CSRA_THREADS = 128;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <bool SIGN, int NB>
__host__ __device__ constexpr size_t csra_warp_smem() {
  return size_t(NB) * 32 * (SIGN ? 4 : 16) + 3 * 512;
}

template <bool SIGN, int NB>
__global__ void __launch_bounds__(CSRA_THREADS)
    csr_step_async_kernel(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                          const int8_t* __restrict__ val, const void* __restrict__ g_cur, void* __restrict__ g_next,
                          float* __restrict__ xs, float* __restrict__ ys, float* __restrict__ ps, int64_t rp,
                          int32_t R, PhaseConsts k, const float* __restrict__ a_rep = nullptr) {
  constexpr int EB = SIGN ? 4 : 16;
  extern __shared__ __align__(16) unsigned char csra_sm[];
  const int lane = threadIdx.x & 31;
  unsigned char* wsm = csra_sm + (threadIdx.x >> 5) * csra_warp_smem<SIGN, NB>();
  const uint32_t slot0 = static_cast<uint32_t>(__cvta_generic_to_shared(wsm)) + lane * EB;
  const float* xyp = reinterpret_cast<const float*>(wsm + NB * 32 * EB);
  const uint32_t xyp0 = static_cast<uint32_t>(__cvta_generic_to_shared(xyp)) + lane * 16;
  const int chunks = static_cast<int>((R + CSR_RCHUNK - 1) / CSR_RCHUNK);
  const int64_t tasks = static_cast<int64_t>(n) * chunks;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t stream = l2::state_policy(), keep = l2::evict_last();
  const uint32_t rsb = static_cast<uint32_t>(rp) * (SIGN ? 1u : 4u);
  for (int64_t t = wid; t < tasks; t += nw) {
    const int i = static_cast<int>(t / chunks);
    const int r = static_cast<int>(t % chunks) * CSR_RCHUNK + 4 * lane;
    const size_t off = static_cast<size_t>(i) * rp + r;
    // this task's x, y, p ride along with the first gather batch
    cp_async16(xyp0, xs + off, stream);
    cp_async16(xyp0 + 512, ys + off, stream);
    cp_async16(xyp0 + 1024, ps + off, stream);
    const int kb = rowptr[i], ke = rowptr[i + 1];
    const char* gb = static_cast<const char*>(g_cur) + static_cast<size_t>(r) * (SIGN ? 1 : 4);
    long long acc[4] = {0, 0, 0, 0};
    for (int k0 = kb; k0 < ke; k0 += 32) {
      const int cnt = min(32, ke - k0);
      int jl = 0, vl = 0;
      if (lane < cnt) {
        jl = col[k0 + lane];
        vl = val[k0 + lane];
      }
      for (int b0 = 0; b0 < cnt; b0 += NB) {
        const int nb = min(NB, cnt - b0);
#pragma unroll
        for (int s = 0; s < NB; ++s) {
          const int j = __shfl_sync(0xffffffffu, jl, b0 + s);
          if (s < nb) {
            const char* src = gb + static_cast<uint64_t>(static_cast<uint32_t>(j)) * rsb;
            if (SIGN)
              cp_async4(slot0 + s * 32 * EB, src, keep);
            else
              cp_async16(slot0 + s * 32 * EB, src, keep);
          }
        }
        cp_async_commit_wait_all();
#pragma unroll
        for (int s = 0; s < NB; ++s) {
          const long long v = __shfl_sync(0xffffffffu, vl, b0 + s);
          if (s < nb) {
            if (SIGN) {
              const char4 g = *reinterpret_cast<const char4*>(wsm + s * 32 * EB + lane * EB);
              acc[0] += v * g.x;
              acc[1] += v * g.y;
              acc[2] += v * g.z;
              acc[3] += v * g.w;
            } else {
              const int4 q = *reinterpret_cast<const int4*>(wsm + s * 32 * EB + lane * EB);
              acc[0] += v * q.x;
              acc[1] += v * q.y;
              acc[2] += v * q.z;
              acc[3] += v * q.w;
            }
          }
        }
      }
    }
    cp_async_commit_wait_all();  // rows without nonzeros: x, y, p still in flight
    float4 x4 = *reinterpret_cast<const float4*>(xyp + 4 * lane);
    float4 y4 = *reinterpret_cast<const float4*>(xyp + 128 + 4 * lane);
    float4 p4 = *reinterpret_cast<const float4*>(xyp + 256 + 4 * lane);
    __syncwarp();  // the next task's cp.async reuses this warp's slots
    if (r >= R) continue;
    float F[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      F[e] = SIGN ? static_cast<float>(acc[e]) : __fmul_rn(__ll2float_rn(acc[e]), 0x1p-30f);
    PhaseConsts kk[4] = {k, k, k, k};
    if (a_rep) {
#pragma unroll
      for (int e = 0; e < 4; ++e) kk[e].a = a_rep[min(r + e, R - 1)];
    }
    gsb_phase(F[0], x4.x, y4.x, p4.x, kk[0]);
    gsb_phase(F[1], x4.y, y4.y, p4.y, kk[1]);
    gsb_phase(F[2], x4.z, y4.z, p4.z, kk[2]);
    gsb_phase(F[3], x4.w, y4.w, p4.w, kk[3]);
    l2::st_f4(xs + off, x4, stream);
    l2::st_f4(ys + off, y4, stream);
    l2::st_f4(ps + off, p4, stream);
    if (SIGN) {
      char4 s;
      s.x = sgn8(x4.x);
      s.y = sgn8(x4.y);
      s.z = sgn8(x4.z);
      s.w = sgn8(x4.w);
      l2::st_u32(static_cast<int8_t*>(g_next) + off, *reinterpret_cast<uint32_t*>(&s), keep);
    } else {
      l2::st_i4(static_cast<int32_t*>(g_next) + off,
                make_int4(quant30(x4.x), quant30(x4.y), quant30(x4.z), quant30(x4.w)), keep);
    }
  }
}

template <bool SIGN, int NB>
inline cudaError_t launch_csr_async(cudaStream_t st, int sms, int32_t n, const int32_t* rowptr, const int32_t* col,
                                    const int8_t* val, const void* g_cur, void* g_next, float* xs, float* ys,
                                    float* ps, int64_t rp, int32_t R, PhaseConsts k, const float* a_rep) {
  constexpr size_t smem = (CSRA_THREADS / 32) * csra_warp_smem<SIGN, NB>();
  static int per_sm = 0;  // resident blocks per SM (shared memory bound), once per instantiation
  if (per_sm == 0) {
    cudaFuncSetAttribute(csr_step_async_kernel<SIGN, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_step_async_kernel<SIGN, NB>, CSRA_THREADS, smem);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
  }
  const int64_t tasks = int64_t(n) * ((R + CSR_RCHUNK - 1) / CSR_RCHUNK);
  const int wpb = CSRA_THREADS / 32;
  const int blocks = int(std::min<int64_t>((tasks + wpb - 1) / wpb, int64_t(sms) * per_sm));
  csr_step_async_kernel<SIGN, NB><<<blocks, CSRA_THREADS, smem, st>>>(n, rowptr, col, val, g_cur, g_next, xs, ys,
                                                                      ps, rp, R, k, a_rep);
  return cudaGetLastError();
}

// B operand of the current (spin-major) state: sign bytes or q = rint(x 2^30).
template <bool SIGN>
__global__ void csr_prep_kernel(const float* __restrict__ xs, void* __restrict__ g, size_t count) {
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < count;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (SIGN)
      static_cast<int8_t*>(g)[idx] = sgn8(xs[idx]);
    else
      static_cast<int32_t*>(g)[idx] = quant30(xs[idx]);
  }
}

// Replica-major [R][ld] <-> spin-major [n][rp] through 32x32 shared tiles.
__global__ void transpose_f32_kernel(const float* __restrict__ src, float* __restrict__ dst, int32_t rows,
                                     int32_t cols, int64_t ld_src, int64_t ld_dst) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    tile[k][threadIdx.x] = (r < rows && c < cols) ? src[static_cast<size_t>(r) * ld_src + c] : 0.0f;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < rows) dst[static_cast<size_t>(c) * ld_dst + r] = tile[threadIdx.x][k];
  }
}

// Readout on CSR from the replica-major state: sign plane + E2[r] = sum_i s_i sum_k val_k s_{col_k}.
constexpr int CSR_RO_THREADS = 512;
__global__ void __launch_bounds__(CSR_RO_THREADS)
    csr_readout_kernel(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const int8_t* __restrict__ val, const float* __restrict__ x, int64_t ld, int32_t R,
                       uint8_t* __restrict__ sign_out, unsigned long long* __restrict__ e2) {
  extern __shared__ float xsm[];
  __shared__ long long red[CSR_RO_THREADS / 32];
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const float v = x[static_cast<size_t>(r) * ld + i];
      xsm[i] = v;
      sign_out[static_cast<size_t>(r) * ld + i] = static_cast<uint8_t>(sgn8(v));
    }
    __syncthreads();
    long long part = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      long long f = 0;
      for (int kk = rowptr[i]; kk < rowptr[i + 1]; ++kk) f += (xsm[col[kk]] >= 0.0f) ? val[kk] : -val[kk];
      part += (xsm[i] >= 0.0f) ? f : -f;
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x < 32) {
      long long sacc = threadIdx.x < CSR_RO_THREADS / 32 ? red[threadIdx.x] : 0;
      for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
      if (threadIdx.x == 0) e2[r] = static_cast<unsigned long long>(sacc);
    }
    __syncthreads();
  }
}

inline int launch_csr_readout(cudaStream_t st, int sms, int32_t n, const int32_t* rowptr, const int32_t* col,
                              const int8_t* val, const float* x, int64_t ld, int32_t R, uint8_t* sign_out,
                              unsigned long long* e2) {
  const size_t smem = sizeof(float) * size_t(n);
  if (smem > 200 * 1024) return int(cudaErrorInvalidValue);
  cudaFuncSetAttribute(csr_readout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  csr_readout_kernel<<<std::min<int>(R, sms * 4), CSR_RO_THREADS, smem, st>>>(n, rowptr, col, val, x, ld, R,
                                                                              sign_out, e2);
  return int(cudaGetLastError());
}

}  // namespace sbg
