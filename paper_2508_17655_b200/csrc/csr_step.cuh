// GSB step for sparse integer couplings (CSR, both triangles, int8 values).
//
// Same semantics as the dense step (engine.cpp:55-110 on the dense view of
// the instance); the field is the exact integer sum
//   sign variants:  F_i = sum_k val_k * sgn(x_{col_k})
//   fixed-point:    F_i = fl32(sum_k val_k * rint(x_{col_k} 2^30)) * 2^-30
// which equals the dense tensor-core field bit for bit (zeros contribute 0).
//
// Layout/strategy: one CTA owns RPB whole replicas; their fp32 x vectors are
// staged once into shared memory (so the gather x[col] is an on-chip random
// read and x_i for the update never re-reads HBM), the CSR arrays stream from
// L2 once per RPB replicas, and each thread updates spins i, i+blockDim, ...
// with coalesced replica-major state accesses. Because a CTA owns its
// replicas entirely, the in-place update has no cross-CTA hazard.
#pragma once

#include <cstdint>

#include "gsb_phase.cuh"

namespace sbg {

constexpr int CSR_THREADS = 512;

template <int RPB, bool SIGN>
__global__ void __launch_bounds__(CSR_THREADS)
    csr_step_kernel(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                    const int8_t* __restrict__ val, float* __restrict__ x, float* __restrict__ y,
                    float* __restrict__ p, int64_t ld, int32_t R, PhaseConsts k) {
  extern __shared__ float xs[];  // [RPB][n]
  for (int rb = blockIdx.x * RPB; rb < R; rb += gridDim.x * RPB) {
    const int nr = min(RPB, R - rb);
    for (int t = 0; t < nr; ++t)
      for (int i = threadIdx.x; i < n; i += blockDim.x) xs[t * n + i] = x[static_cast<size_t>(rb + t) * ld + i];
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      long long acc[RPB];
#pragma unroll
      for (int t = 0; t < RPB; ++t) acc[t] = 0;
      const int kb = rowptr[i], ke = rowptr[i + 1];
      for (int kk = kb; kk < ke; ++kk) {
        const int j = col[kk];
        const int v = val[kk];
#pragma unroll
        for (int t = 0; t < RPB; ++t) {
          const float xj = xs[t * n + j];
          if (SIGN)
            acc[t] += (xj >= 0.0f) ? v : -v;
          else
            acc[t] += static_cast<long long>(v) * quant30(xj);
        }
      }
#pragma unroll
      for (int t = 0; t < RPB; ++t) {
        if (t < nr) {
          const size_t off = static_cast<size_t>(rb + t) * ld + i;
          const float F = SIGN ? static_cast<float>(acc[t]) : __fmul_rn(__ll2float_rn(acc[t]), 0x1p-30f);
          float xi = xs[t * n + i], yi = y[off], pi = p[off];
          gsb_phase(F, xi, yi, pi, k);
          x[off] = xi;
          y[off] = yi;
          p[off] = pi;
        }
      }
    }
    __syncthreads();
  }
}

// Readout on CSR: sign plane + E2[r] = sum_i s_i sum_k val_k s_{col_k}.
__global__ void __launch_bounds__(CSR_THREADS)
    csr_readout_kernel(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                       const int8_t* __restrict__ val, const float* __restrict__ x, int64_t ld, int32_t R,
                       uint8_t* __restrict__ sign_out, unsigned long long* __restrict__ e2) {
  extern __shared__ float xs[];
  __shared__ long long red[CSR_THREADS / 32];
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const float v = x[static_cast<size_t>(r) * ld + i];
      xs[i] = v;
      sign_out[static_cast<size_t>(r) * ld + i] = static_cast<uint8_t>(sgn8(v));
    }
    __syncthreads();
    long long part = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      long long f = 0;
      for (int kk = rowptr[i]; kk < rowptr[i + 1]; ++kk) f += (xs[col[kk]] >= 0.0f) ? val[kk] : -val[kk];
      part += (xs[i] >= 0.0f) ? f : -f;
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x < 32) {
      long long s = threadIdx.x < CSR_THREADS / 32 ? red[threadIdx.x] : 0;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (threadIdx.x == 0) e2[r] = static_cast<unsigned long long>(s);
    }
    __syncthreads();
  }
}

inline int csr_rpb(int32_t n) { return (2 * sizeof(float) * size_t(n) <= 200 * 1024) ? 2 : 1; }

inline int launch_csr_step(cudaStream_t st, int sms, int32_t n, const int32_t* rowptr, const int32_t* col,
                           const int8_t* val, float* x, float* y, float* p, int64_t ld, int32_t R, bool sign,
                           PhaseConsts k, uint64_t M, uint64_t m) {
  k.inv = 1.0f / static_cast<float>(M - m);  // host: IEEE division == __frcp_rn
  const int rpb = csr_rpb(n);
  const size_t smem = sizeof(float) * size_t(n) * rpb;
  if (smem > 227 * 1024) return int(cudaErrorInvalidValue);
  const int blocks = std::min<int>((R + rpb - 1) / rpb, sms * 4);
#define SBG_CSR_LAUNCH(RPB_, SIGN_)                                                                     \
  do {                                                                                                  \
    auto kern = csr_step_kernel<RPB_, SIGN_>;                                                           \
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));                 \
    kern<<<blocks, CSR_THREADS, smem, st>>>(n, rowptr, col, val, x, y, p, ld, R, k);                    \
  } while (0)
  if (rpb == 2) {
    if (sign) SBG_CSR_LAUNCH(2, true); else SBG_CSR_LAUNCH(2, false);
  } else {
    if (sign) SBG_CSR_LAUNCH(1, true); else SBG_CSR_LAUNCH(1, false);
  }
#undef SBG_CSR_LAUNCH
  return int(cudaGetLastError());
}

inline int launch_csr_readout(cudaStream_t st, int sms, int32_t n, const int32_t* rowptr, const int32_t* col,
                              const int8_t* val, const float* x, int64_t ld, int32_t R, uint8_t* sign_out,
                              unsigned long long* e2) {
  const size_t smem = sizeof(float) * size_t(n);
  if (smem > 200 * 1024) return int(cudaErrorInvalidValue);
  cudaFuncSetAttribute(csr_readout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  csr_readout_kernel<<<std::min<int>(R, sms * 4), CSR_THREADS, smem, st>>>(n, rowptr, col, val, x, ld, R,
                                                                           sign_out, e2);
  return int(cudaGetLastError());
}

}  // namespace sbg
