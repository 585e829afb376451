// GSB step for dense integer couplings on the 5th-gen tensor cores.
//
// One launch = one time step of every replica (sbopt::step,
// /root/reference/proj/core/src/engine.cpp:55-110, batched over R):
//
//   F[i, r] = sum_j J[i, j] * G[r, j]          tcgen05.mma kind::i8, s32 in TMEM
//   (x, y, p)[r, i] <- phase(F[i, r], ...)     fused epilogue (gsb_phase.cuh)
//   G'[r, i] <- sgn(x) or fixed-point planes   written for the next launch
//
// G is the MMA B operand, K-major: G[r][j] int8, one plane (dsb/gdsb: the
// sign matrix, exact +-1) or four byte planes of q = rint(x * 2^30)
// (bsb/gbsb: signed base-256 digits, qdigits; the field sum is then exact in integers and scaled
// once). J is the A operand, row-major int8 [npad][npad]. Both arrive by TMA
// (128-byte swizzle) into a STAGES-deep mbarrier ring; one elected lane of
// warp 1 issues the MMAs into one of two TMEM accumulator buffers, so the
// epilogue of tile t (8 warps, tcgen05.ld -> registers) overlaps the MMA of
// tile t+1. CTAs are persistent over a static round-robin tile schedule.
//
// The state is replica-major fp32 [rpad][ld] (ld = npad): a warp's 32 lanes
// are 32 consecutive spins i of one replica, so every state access is one
// fully-used 128-byte line per (replica, array).
//
// Modes: Step (the hot path), Readout (E2[r] = sum_i s_i (J s)_i, the
// ising_energy of model.cpp:112-123, reduced with warp shuffles + one int64
// atomic per warp and column), Fields (teacher-forced field dump for parity).
#pragma once

#include <cstdint>
#include <cuda.h>

#include "gsb_phase.cuh"
#include "ptx.cuh"

namespace sbg {

enum class EpiMode : int { Step = 0, Readout = 1, Fields = 2 };

struct StepArgs {
  int32_t n, npad, R, rpad;
  int32_t num_m, num_n;
  int64_t ld;
  float* x;
  float* y;
  float* p;
  uint8_t* planes_next;       // Step: [NPLANES][rpad][npad]
  int8_t* sign_out;           // Step (planes mode, optional): [rpad][npad]
  const int8_t* sign_in;      // Readout: [rpad][npad]
  unsigned long long* e2;     // Readout: [R], two's complement int64 sums
  void* fields_out;           // Fields: int32 (sign) or float (planes) [rpad][ld]
  PhaseConsts k;              // a, c, dt; inv filled in-kernel
  const uint64_t* m_dev;      // step index base in device memory (graph replay)
  int64_t m_off;              // m = (m_dev ? *m_dev : 0) + m_off
  uint64_t M;                 // total steps
  int32_t dbg;                // dev experiments: 1 = no state traffic, 2 = no MMA (F = 0)
  int32_t a_unsigned;         // A operand bytes are u8 (low planes of a fixed-point J)
  int32_t kpad;               // K extent (global padded n; == npad unless row-sharded)
  int64_t sign_ld;            // Readout: row pitch of sign_in (sign_in may point into a wider G)
};

template <int NPLANES, int BN>
struct StepCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 128;                       // bytes of K per stage
  static constexpr int A_BYTES = BM * BK;              // 16 KB
  static constexpr int B_PLANE_BYTES = BN * BK;
  static constexpr int STAGE_BYTES = A_BYTES + NPLANES * B_PLANE_BYTES;
  static constexpr int STAGES = (196608 / STAGE_BYTES) < 8 ? (196608 / STAGE_BYTES) : 8;
  static constexpr int ACC_COLS = NPLANES * BN;        // one accumulator buffer
  static constexpr int TMEM_COLS = 2 * ACC_COLS;       // double buffered
  static constexpr int CW = NPLANES == 1 ? 32 : 16;    // epilogue column chunk
  static constexpr int THREADS = 384;                  // 4 control + 8 epilogue warps
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static_assert(TMEM_COLS == 32 || TMEM_COLS == 64 || TMEM_COLS == 128 || TMEM_COLS == 256 ||
                    TMEM_COLS == 512,
                "TMEM allocation must be a power of two <= 512 columns");
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  static_assert((BN / 2) % CW == 0, "epilogue half must be a multiple of the chunk");
  static_assert(STAGES >= 2, "pipeline depth");
};

template <int CW>
__device__ __forceinline__ void tmem_ld_chunk(uint32_t taddr, uint32_t (&v)[CW]);

template <>
__device__ __forceinline__ void tmem_ld_chunk<32>(uint32_t taddr, uint32_t (&v)[32]) {
  ptx::tmem_ld32(taddr, v);
}

template <>
__device__ __forceinline__ void tmem_ld_chunk<16>(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

template <int NPLANES, int BN, EpiMode MODE>
__global__ void __launch_bounds__(384, 1)
    gsb_step_i8_kernel(const __grid_constant__ CUtensorMap tmJ, const __grid_constant__ CUtensorMap tmG,
                       const StepArgs args) {
  using Cfg = StepCfg<NPLANES, BN>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int CW = Cfg::CW;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;  // 128B swizzle wants 1024B-aligned tiles
  uint8_t* smem = smem_raw + (base - raw_addr);
  const uint32_t a_base = base;
  const uint32_t b_base = base + STAGES * Cfg::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  auto full_bar = [&](int s) { return ptx::smem_u32(bars + s); };
  auto empty_bar = [&](int s) { return ptx::smem_u32(bars + STAGES + s); };
  auto tfull_bar = [&](int b) { return ptx::smem_u32(bars + 2 * STAGES + b); };
  auto tempty_bar = [&](int b) { return ptx::smem_u32(bars + 2 * STAGES + 2 + b); };

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), 1);
      ptx::mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(tfull_bar(b), 1);
      ptx::mbar_init(tempty_bar(b), 8);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc(ptx::smem_u32(tmem_slot), Cfg::TMEM_COLS);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = args.num_m * args.num_n;
  const int KB = (args.kpad ? args.kpad : args.npad) / Cfg::BK;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      ptx::prefetch_tmap(&tmJ);
      ptx::prefetch_tmap(&tmG);
      int stage = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m_blk = t % args.num_m;
        const int n_blk = t / args.num_m;
        for (int kb = 0; kb < KB; ++kb) {
          ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
          ptx::mbar_arrive_expect_tx(full_bar(stage), Cfg::STAGE_BYTES);
          ptx::tma_load_2d(a_base + stage * Cfg::A_BYTES, &tmJ, full_bar(stage), kb * Cfg::BK,
                           m_blk * Cfg::BM);
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl) {
            ptx::tma_load_2d(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES, &tmG, full_bar(stage),
                             kb * Cfg::BK, pl * args.rpad + n_blk * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t idesc_s = ptx::idesc_i8(128, BN, !args.a_unsigned, true);
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        const int buf = lt & 1;
        const uint32_t use_ph = (lt >> 1) & 1;
        ptx::mbar_wait(tempty_bar(buf), use_ph ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_base = tmem_base + buf * Cfg::ACC_COLS;
        for (int kb = 0; kb < KB; ++kb) {
          ptx::mbar_wait(full_bar(stage), ph);
          ptx::tc_fence_after();
          const uint64_t adesc = ptx::smem_desc_k_sw128(a_base + stage * Cfg::A_BYTES);
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl) {
            const uint64_t bdesc =
                ptx::smem_desc_k_sw128(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES);
            const uint32_t idesc = idesc_s;  // sign plane or signed digit planes (qdigits)
#pragma unroll
            for (int k = 0; k < Cfg::BK / 32; ++k) {
              // +32 bytes along K inside the 128-byte swizzle atom = +2 in the
              // descriptor's 16-byte start-address field.
              ptx::mma_i8(d_base + pl * BN, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            }
          }
          ptx::mma_commit(empty_bar(stage));
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
        ptx::mma_commit(tfull_bar(buf));
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int q = warp & 3;           // TMEM lane quadrant this warp may access
    const int h = (warp - 4) >> 2;    // column half
    PhaseConsts k = args.k;
    if (MODE == EpiMode::Step) {
      const uint64_t m = (args.m_dev ? *args.m_dev : 0ull) + static_cast<uint64_t>(args.m_off);
      k.inv = __frcp_rn(static_cast<float>(args.M - m));
    }
    const size_t plane_stride = static_cast<size_t>(args.rpad) * args.npad;
    int lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      const int m_blk = t % args.num_m;
      const int n_blk = t / args.num_m;
      const int buf = lt & 1;
      const uint32_t use_ph = (lt >> 1) & 1;
      ptx::mbar_wait(tfull_bar(buf), use_ph);
      __syncwarp();
      ptx::tc_fence_after();
      const int row = m_blk * 128 + q * 32 + lane;
      const bool row_ok = row < args.n;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * Cfg::ACC_COLS;
#pragma unroll 1
      for (int c0 = h * (BN / 2); c0 < (h + 1) * (BN / 2); c0 += CW) {
        const int r0 = n_blk * BN + c0;
        // ---- accumulator chunk -> registers -> field values
        float F[CW];
        int32_t Fi[CW];
        if (NPLANES == 1) {
          uint32_t v[CW];
          tmem_ld_chunk<CW>(t_row + c0, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            Fi[j] = static_cast<int32_t>(v[j]);
            F[j] = static_cast<float>(Fi[j]);
          }
        } else {
          long long tot[CW];
#pragma unroll
          for (int j = 0; j < CW; ++j) tot[j] = 0;
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl) {
            uint32_t v[CW];
            tmem_ld_chunk<CW>(t_row + pl * BN + c0, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CW; ++j)
              tot[j] += static_cast<long long>(static_cast<int32_t>(v[j])) << (8 * pl);
          }
#pragma unroll
          for (int j = 0; j < CW; ++j) F[j] = __fmul_rn(__ll2float_rn(tot[j]), 0x1p-30f);
        }
        if (r0 >= args.R) continue;  // padded replica columns are inert
        if (MODE == EpiMode::Step) {
          if (row_ok) {
            float xs[CW], ys[CW], ps[CW];
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              const size_t off = static_cast<size_t>(r0 + j) * args.ld + row;
              if (r0 + j < args.R) {
                xs[j] = args.x[off];
                ys[j] = args.y[off];
                ps[j] = args.p[off];
              }
            }
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              if (r0 + j < args.R) {
                const size_t off = static_cast<size_t>(r0 + j) * args.ld + row;
                gsb_phase(F[j], xs[j], ys[j], ps[j], k);
                args.x[off] = xs[j];
                args.y[off] = ys[j];
                args.p[off] = ps[j];
                const size_t goff = static_cast<size_t>(r0 + j) * args.npad + row;
                if (NPLANES == 1) {
                  args.planes_next[goff] = static_cast<uint8_t>(sgn8(xs[j]));
                } else {
                  const uint32_t qv = qdigits(quant30(xs[j]));
#pragma unroll
                  for (int pl = 0; pl < NPLANES; ++pl)
                    args.planes_next[pl * plane_stride + goff] = static_cast<uint8_t>(qv >> (8 * pl));
                  if (args.sign_out) args.sign_out[goff] = sgn8(xs[j]);
                }
              }
            }
          }
        } else if (MODE == EpiMode::Readout) {
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            long long part = 0;
            if (row_ok && r0 + j < args.R) {
              const int s = args.sign_in[static_cast<size_t>(r0 + j) * (args.sign_ld ? args.sign_ld : args.npad) + row];
              part = static_cast<long long>(s) * Fi[j];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (lane == 0 && r0 + j < args.R)
              atomicAdd(args.e2 + (r0 + j), static_cast<unsigned long long>(part));
          }
        } else {  // Fields
          if (row_ok) {
#pragma unroll
            for (int j = 0; j < CW; ++j) {
              if (r0 + j < args.R) {
                const size_t off = static_cast<size_t>(r0 + j) * args.ld + row;
                if (NPLANES == 1)
                  static_cast<int32_t*>(args.fields_out)[off] = Fi[j];
                else
                  static_cast<float*>(args.fields_out)[off] = F[j];
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(tempty_bar(buf));
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
}

}  // namespace sbg

