// Extreme eigenvalues of the coupling matrix on the device: the numerical branch
// of auto_tune (spectral.cpp:207-246, :294-326) without materialising fp64 J.
//
//  * n == 2: closed form (spectral.cpp:121-138); 3 <= n <= 32: cyclic Jacobi
//    (:140-198) in one warp -- each rotation's three k-loops touch disjoint
//    elements per k, so lane k doing element k is the serial loop reordered
//    without changing any operation.
//  * n > 32: shifted power iteration (:50-118) as ONE cooperative persistent
//    kernel. Per iteration: J v over the whole grid (8 lanes per row, the
//    row_dot lane/tail/combine order of kernels.hpp:14-30, so J v is bitwise the
//    reference's for any J the device holds exactly: int8 and CSR int8), then the
//    reference's sequential reductions (dot, residual, ||w||, norm2 -- one running
//    sum each, kept serial so every rounding matches) and its stall/perturbation
//    logic (Xoshiro256pp(0xB1F0CA7E), perturbation cap 4, stall window
//    max(64, n/4)) on CTA 0, then the update v <- w/||w|| over the grid.
//    All fp64 arithmetic uses explicit _rn intrinsics (no contraction), matching
//    the reference built with -ffp-contract=off.
#pragma once

#include <cstdint>

#include "aux_kernels.cuh"

namespace sbg {

enum { JV_DENSE_I8 = 1, JV_CSR_I8 = 2, JV_DENSE_FX = 3 };

struct JView {
  int kind;
  int64_t n, ld;                 // dense: row stride in bytes
  const int8_t* J;               // dense int8, or byte plane 0 of the fixed-point image
  int64_t plane;                 // fixed point: bytes between planes
  double scale;                  // fixed point: 2^-s
  const int32_t* rowptr;         // CSR
  const int32_t* col;
  const int8_t* val;

  __device__ __forceinline__ double at(int64_t i, int64_t j) const {  // dense kinds
    if (kind == JV_DENSE_I8) return double(J[i * ld + j]);
    const uint8_t* b = reinterpret_cast<const uint8_t*>(J) + i * ld + j;
    const int32_t q = int32_t(b[0]) | (int32_t(b[plane]) << 8) | (int32_t(int8_t(b[2 * plane])) * 65536);
    return __dmul_rn(double(q), scale);
  }
};

// out_i = row_dot(J_i, v) in the lane order of kernels.hpp:14-30, computed by the 8
// consecutive lanes l = threadIdx.x & 7; the result is valid in lane 0 of the group.
// Called by all 32 lanes of the warp (shuffles); groups with live == false add nothing.
__device__ __forceinline__ double row_dot8(const JView& J, int64_t i, const double* __restrict__ v, int l, bool live) {
  const int64_t n = J.n, n8 = n & ~int64_t(7);
  double acc = 0.0;
  if (!live) {
  } else if (J.kind == JV_CSR_I8) {
    for (int32_t k = J.rowptr[i]; k < J.rowptr[i + 1]; ++k) {
      const int64_t c = J.col[k];
      if ((c < n8 ? int(c & 7) : 0) == l) acc = __dadd_rn(acc, __dmul_rn(double(J.val[k]), v[c]));
    }
  } else {
    for (int64_t j = l; j < n8; j += 8) acc = __dadd_rn(acc, __dmul_rn(J.at(i, j), v[j]));
    if (l == 0)
      for (int64_t j = n8; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(J.at(i, j), v[j]));
  }
  acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));  // (a0+a1), (a2+a3), ...
  acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));  // (a0+a1)+(a2+a3), ...
  acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
  return acc;
}

// Per-row sum of squares (off-diagonal) and of absolute values: offdiagonal_sigma
// (spectral.cpp:254-266) and gershgorin_bound (:30-38). One warp per row.
__global__ void row_stats_kernel(JView J, double* __restrict__ sumsq, double* __restrict__ abssum) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < J.n; i += warps) {
    double sq = 0.0, ab = 0.0;
    if (J.kind == JV_CSR_I8) {
      for (int32_t k = J.rowptr[i] + lane; k < J.rowptr[i + 1]; k += 32) {
        const double x = double(J.val[k]);
        sq = __dadd_rn(sq, __dmul_rn(x, x));
        ab = __dadd_rn(ab, fabs(x));
      }
    } else {
      for (int64_t j = lane; j < J.n; j += 32) {
        const double x = J.at(i, j);
        if (j != i) sq = __dadd_rn(sq, __dmul_rn(x, x));
        ab = __dadd_rn(ab, fabs(x));
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
      ab = __dadd_rn(ab, __shfl_xor_sync(0xffffffffu, ab, o));
    }
    if (lane == 0) {
      sumsq[i] = sq;
      abssum[i] = ab;
    }
  }
}

// ------------------------------------------------------------------ n <= 32

// out: [0] lambda_max, [1] lambda_min, [2..2+n) v_max, [2+n..2+2n) v_min.
__global__ void __launch_bounds__(32) spectral_small_kernel(JView J, double* __restrict__ out) {
  __shared__ double a[32 * 32], V[32 * 32];
  __shared__ double bc[1];
  __shared__ int ext[2];
  const int n = int(J.n), k = threadIdx.x;
  if (n == 2) {  // spectral.cpp:121-138
    if (k == 0) {
      const double c01 = J.kind == JV_CSR_I8 ? (J.rowptr[1] > J.rowptr[0] ? double(J.val[J.rowptr[0]]) : 0.0)
                                             : J.at(0, 1);
      const double mag = fabs(c01), s = __ddiv_rn(1.0, __dsqrt_rn(2.0));
      out[0] = mag;
      out[1] = -mag;
      out[2] = s;
      out[3] = c01 >= 0.0 ? s : -s;
      out[4] = s;
      out[5] = c01 >= 0.0 ? -s : s;
    }
    return;
  }
  for (int r = 0; r < n; ++r)
    if (k < n) {
      a[r * n + k] = 0.0;
      V[r * n + k] = r == k ? 1.0 : 0.0;
    }
  __syncwarp();
  if (k < n) {
    if (J.kind == JV_CSR_I8) {
      for (int32_t q = J.rowptr[k]; q < J.rowptr[k + 1]; ++q) a[k * n + J.col[q]] = double(J.val[q]);
    } else {
      for (int j = 0; j < n; ++j) a[k * n + j] = J.at(k, j);
    }
  }
  __syncwarp();
  for (int sweep = 0; sweep < 64; ++sweep) {
    if (k == 0) {
      double off = 0.0;
      for (int p = 0; p < n; ++p)
        for (int q = p + 1; q < n; ++q) off = __dadd_rn(off, __dmul_rn(a[p * n + q], a[p * n + q]));
      bc[0] = off;
    }
    __syncwarp();
    if (bc[0] < 1e-28) break;
    for (int p = 0; p < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double theta = __ddiv_rn(__dsub_rn(a[q * n + q], a[p * n + p]), __dmul_rn(2.0, apq));
        const double t = __ddiv_rn(theta >= 0.0 ? 1.0 : -1.0,
                                   __dadd_rn(fabs(theta), __dsqrt_rn(__dadd_rn(__dmul_rn(theta, theta), 1.0))));
        const double cr = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(__dmul_rn(t, t), 1.0)));
        const double sr = __dmul_rn(t, cr);
        __syncwarp();
        if (k < n) {
          const double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = __dsub_rn(__dmul_rn(cr, akp), __dmul_rn(sr, akq));
          a[k * n + q] = __dadd_rn(__dmul_rn(sr, akp), __dmul_rn(cr, akq));
        }
        __syncwarp();
        if (k < n) {
          const double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = __dsub_rn(__dmul_rn(cr, apk), __dmul_rn(sr, aqk));
          a[q * n + k] = __dadd_rn(__dmul_rn(sr, apk), __dmul_rn(cr, aqk));
          const double vkp = V[k * n + p], vkq = V[k * n + q];
          V[k * n + p] = __dsub_rn(__dmul_rn(cr, vkp), __dmul_rn(sr, vkq));
          V[k * n + q] = __dadd_rn(__dmul_rn(sr, vkp), __dmul_rn(cr, vkq));
        }
        __syncwarp();
      }
    }
    __syncwarp();
  }
  __syncwarp();
  if (k == 0) {
    int imax = 0, imin = 0;
    for (int i = 1; i < n; ++i) {
      if (a[i * n + i] > a[imax * n + imax]) imax = i;
      if (a[i * n + i] < a[imin * n + imin]) imin = i;
    }
    ext[0] = imax;
    ext[1] = imin;
    out[0] = a[imax * n + imax];
    out[1] = a[imin * n + imin];
  }
  __syncwarp();
  const int imax = ext[0], imin = ext[1];
  if (k < n) {
    out[2 + k] = V[k * n + imax];
    out[2 + n + k] = V[k * n + imin];
  }
}

// ------------------------------------------------------------------ n > 32

enum { PI_UPDATE = 0, PI_PERTURB = 1, PI_EXIT = 2 };

constexpr int PI_THREADS = 256;
constexpr int PI_CHUNK = 2048;         // elements per staged chunk of the serial reductions
constexpr int PI_V_SMEM = 12288;       // v staged in shared memory for J v up to this n
constexpr int PI_SMEM_BYTES = PI_V_SMEM * 8;  // >= 2 buffers x (v, jv) x PI_CHUNK x 8 B

struct PowerArgs {
  JView J;
  double beta, sign, tol, v_init;
  uint64_t max_iters;
  double* v[2];                  // n each: current / next iterate
  double* jv;                    // n
  unsigned long long* bar;       // grid barrier counter (zero on entry)
  int* ctrl;                     // broadcast of CTA 0's decision
  double* result;                // [0] lambda [1] residual [2] iterations [3] converged [4] final v buffer
};

__device__ __forceinline__ void grid_sync(unsigned long long* bar, unsigned long long& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1ull);
    unsigned long long seen;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(bar) : "memory");
    } while (seen < target);
  }
  __syncthreads();
}

// One pass of the serial reductions over (v, jv), staged through shared memory in
// double-buffered chunks: warps 2.. load chunk k+1 while thread 0 (and thread 32)
// run their running sums over chunk k. f0 / f1 are the per-element chain updates.
template <class F0, class F1>
__device__ __forceinline__ void staged_pass(const double* __restrict__ v, const double* __restrict__ jv, int64_t n,
                                            double* sm, F0&& f0, F1&& f1) {
  const int warp = threadIdx.x >> 5;
  const int ltid = threadIdx.x - 64, nload = PI_THREADS - 64;
  auto stage = [&](int64_t base, int b) {
    double* sv = sm + b * 2 * PI_CHUNK;
    double* sj = sv + PI_CHUNK;
    const int64_t cnt = n - base < PI_CHUNK ? n - base : PI_CHUNK;
    for (int64_t i = ltid; i < cnt; i += nload) {
      sv[i] = v[base + i];
      sj[i] = jv[base + i];
    }
  };
  if (warp >= 2) stage(0, 0);
  __syncthreads();
  for (int64_t base = 0, k = 0; base < n; base += PI_CHUNK, ++k) {
    const int b = int(k & 1);
    if (warp >= 2 && base + PI_CHUNK < n) stage(base + PI_CHUNK, b ^ 1);
    const int64_t cnt = n - base < PI_CHUNK ? n - base : PI_CHUNK;
    const double* sv = sm + b * 2 * PI_CHUNK;
    const double* sj = sv + PI_CHUNK;
    if (threadIdx.x == 0) {
#pragma unroll 8
      for (int64_t i = 0; i < cnt; ++i) f0(sv[i], sj[i]);
    } else if (threadIdx.x == 32) {
#pragma unroll 8
      for (int64_t i = 0; i < cnt; ++i) f1(sv[i], sj[i]);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(PI_THREADS, 1) power_iteration_kernel(PowerArgs A) {
  extern __shared__ __align__(16) double sm[];
  const int64_t n = A.J.n;
  const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const int64_t nthr = int64_t(gridDim.x) * blockDim.x;
  unsigned long long target = 0;
  __shared__ double s_lambda, s_res, s_nw, s_nv;
  __shared__ int s_ctrl;
  for (int64_t i = tid; i < n; i += nthr) A.v[0][i] = A.v_init;
  grid_sync(A.bar, target);

  // CTA 0 / thread 0 state (spectral.cpp:55-60)
  Xoshiro rng(0xB1F0CA7Eull);
  int perturbations = 0;
  double best_residual = __longlong_as_double(0x7ff0000000000000ll);
  uint64_t best_iteration = 0;
  const uint64_t stall_window = uint64_t(n / 4) > 64 ? uint64_t(n / 4) : 64;
  const double conv_bound = __dmul_rn(A.tol, A.beta);
  const double null_bound = __dmul_rn(A.beta, 1e-14);
  const bool v_in_smem = n <= PI_V_SMEM;

  int cur = 0;
  for (uint64_t iter = 1; iter <= A.max_iters; ++iter) {
    const double* __restrict__ vc = A.v[cur];
    double* __restrict__ vn = A.v[cur ^ 1];
    // ---- J v over the grid (v from shared memory when it fits)
    const double* vsrc = vc;
    if (v_in_smem) {
      for (int64_t i = threadIdx.x; i < n; i += PI_THREADS) sm[i] = vc[i];
      __syncthreads();
      vsrc = sm;
    }
    for (int64_t base = (tid >> 5) << 2; base < n; base += (nthr >> 5) << 2) {  // 4 rows per warp
      const int64_t g = base + ((threadIdx.x & 31) >> 3);
      const double r = row_dot8(A.J, g, vsrc, int(threadIdx.x & 7), g < n);
      if ((threadIdx.x & 7) == 0 && g < n) A.jv[g] = r;
    }
    grid_sync(A.bar, target);

    // ---- CTA 0: the reference's serial reductions and control logic
    if (blockIdx.x == 0) {
      double lam = 0.0, nw = 0.0;
      const double sign = A.sign, beta = A.beta;
      // dot(v, jv) (spectral.cpp:21-25) || ||w||^2 of w = sign*jv + beta*v (:99-104, speculative)
      staged_pass(vc, A.jv, n, sm,
                  [&](double v, double j) { lam = __dadd_rn(lam, __dmul_rn(v, j)); },
                  [&](double v, double j) {
                    const double w = __dadd_rn(__dmul_rn(sign, j), __dmul_rn(beta, v));
                    nw = __dadd_rn(nw, __dmul_rn(w, w));
                  });
      if (threadIdx.x == 0) s_lambda = lam;
      if (threadIdx.x == 32) s_nw = __dsqrt_rn(nw);
      __syncthreads();
      const double lambda = s_lambda;
      double res = 0.0;  // ||jv - lambda v|| (:68-73)
      staged_pass(vc, A.jv, n, sm,
                  [&](double v, double j) {
                    const double r = __dsub_rn(j, __dmul_rn(lambda, v));
                    res = __dadd_rn(res, __dmul_rn(r, r));
                  },
                  [](double, double) {});
      if (threadIdx.x == 0) {
        res = __dsqrt_rn(res);
        A.result[0] = lambda;
        A.result[1] = res;
        A.result[2] = double(iter);
        A.result[4] = double(cur);
        int ctrl;
        if (res <= conv_bound) {
          A.result[3] = 1.0;
          ctrl = PI_EXIT;
        } else if (res < __dmul_rn(best_residual, 0.999)) {
          best_residual = res;
          best_iteration = iter;
          ctrl = s_nw <= null_bound ? PI_PERTURB : PI_UPDATE;
        } else if (iter - best_iteration > stall_window && perturbations < 4) {
          ctrl = PI_PERTURB;
          best_iteration = iter;
          best_residual = __longlong_as_double(0x7ff0000000000000ll);
        } else {
          ctrl = s_nw <= null_bound ? PI_PERTURB : PI_UPDATE;
        }
        if (ctrl == PI_PERTURB) {  // :84-93 / :105-111: v += 0.05 U(-1,1), then v /= norm2(v)
          ++perturbations;
          double nv = 0.0;
          for (int64_t i = 0; i < n; ++i) {
            const double u = __dsub_rn(__dmul_rn(2.0, __dmul_rn(double(rng.next() >> 11), 0x1.0p-53)), 1.0);
            const double x = __dadd_rn(vc[i], __dmul_rn(0.05, u));
            vn[i] = x;
            nv = __dadd_rn(nv, __dmul_rn(x, x));
          }
          s_nv = __dsqrt_rn(nv);
        }
        s_ctrl = ctrl;
        *A.ctrl = ctrl;
      }
      __syncthreads();
      if (s_ctrl == PI_PERTURB) {
        for (int64_t i = threadIdx.x; i < n; i += PI_THREADS) vn[i] = __ddiv_rn(vn[i], s_nv);
      } else if (s_ctrl == PI_UPDATE) {  // v <- w / ||w||
        const double nwv = s_nw;
        for (int64_t i = threadIdx.x; i < n; i += PI_THREADS)
          vn[i] = __ddiv_rn(__dadd_rn(__dmul_rn(sign, A.jv[i]), __dmul_rn(beta, vc[i])), nwv);
      }
    }
    grid_sync(A.bar, target);
    if (*reinterpret_cast<volatile int*>(A.ctrl) == PI_EXIT) break;
    cur ^= 1;
  }
}

}  // namespace sbg
