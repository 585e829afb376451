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
// (bsb/gbsb: u8,u8,u8,s8; the field sum is then exact in integers and scaled
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
  PhaseConsts k;              // a, c, dt; denom filled in-kernel
  const uint64_t* m_dev;      // step index base in device memory (graph replay)
  int64_t m_off;              // m = (m_dev ? *m_dev : 0) + m_off
  uint64_t M;                 // total steps
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
  const int KB = args.npad / Cfg::BK;

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
      constexpr uint32_t idesc_s = ptx::idesc_i8(128, BN, true, true);
      constexpr uint32_t idesc_u = ptx::idesc_i8(128, BN, true, false);
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
            const uint32_t idesc = (NPLANES == 1 || pl == NPLANES - 1) ? idesc_s : idesc_u;
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
      k.denom = static_cast<float>(args.M - m);
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
                  const uint32_t qv = static_cast<uint32_t>(quant30(xs[j]));
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
              const int s = args.sign_in[static_cast<size_t>(r0 + j) * args.npad + row];
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

namespace sbg {

// ---------------------------------------------------------------------------
// Step mode, TMA-staged state (the hot path).
//
// Same operand pipeline and MMA as above; the epilogue no longer gathers the
// fp32 state with per-thread loads. Instead a loader warp streams x, y, p
// chunks (128 spins x CW replicas each) from HBM into a NBUF-deep shared-memory
// ring with TMA, the 8 epilogue warps update them in place from the TMEM
// accumulator (shared-memory reads/writes are conflict-free: lanes are
// consecutive spins), and a storer warp writes x, y, p and the next B operand
// (sign plane or fixed-point planes) back with TMA stores. Tensor-map bounds
// (n spins x R replicas) zero-fill loads and clip stores at the edges, so the
// epilogue carries no predicates. HBM sees exactly 12 B read + 12 B written
// per spin-update plus the 1 (sign) / 4 (planes) bytes of the next operand.
// ---------------------------------------------------------------------------

template <int NPLANES, int BN>
struct TmaStepCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 128;
  static constexpr int A_BYTES = BM * BK;
  static constexpr int B_PLANE_BYTES = BN * BK;
  static constexpr int STAGE_BYTES = A_BYTES + NPLANES * B_PLANE_BYTES;
  static constexpr int STAGES = NPLANES == 1 ? 3 : 2;
  static constexpr int CW = 16;                         // replicas per state chunk
  static constexpr int CWH = CW / 2;                    // per epilogue thread (two column halves)
  static constexpr int NBUF = NPLANES == 1 ? 4 : 3;
  static constexpr int ST_ARR = CW * BM * 4;            // one fp32 array chunk: 8 KB
  static constexpr int ST_G = CW * BM;                  // one byte plane chunk: 2 KB
  static constexpr int BUF_RAW = 3 * ST_ARR + NPLANES * ST_G;
  static constexpr int BUF_BYTES = (BUF_RAW + 1023) / 1024 * 1024;
  static constexpr int ACC_COLS = NPLANES * BN;
  static constexpr int TMEM_COLS = 2 * ACC_COLS;
  static constexpr int THREADS = 384;
  static constexpr int NUM_BARS = 2 * STAGES + 4 + 3 * NBUF;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + NBUF * BUF_BYTES + 1024 + 8 * NUM_BARS + 64;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(BN % CW == 0, "chunking");
  static_assert(TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation");
};

struct TmaMaps {
  CUtensorMap J;       // A operand, int8 [npad][npad], 128B swizzle
  CUtensorMap Gin;     // B operand in, [NPLANES*rpad][npad], 128B swizzle
  CUtensorMap Gout;    // B operand out, [rows][n] (sign: R rows; planes: NPLANES*rpad), no swizzle
  CUtensorMap X, Y, P; // fp32 state [R][n] (row pitch ld), no swizzle
};

template <int NPLANES, int BN>
__global__ void __launch_bounds__(384, 1)
    gsb_step_tma_kernel(const __grid_constant__ TmaMaps maps, const StepArgs args) {
  using Cfg = TmaStepCfg<NPLANES, BN>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int NBUF = Cfg::NBUF;
  constexpr int CW = Cfg::CW;
  constexpr int CWH = Cfg::CWH;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_addr);
  const uint32_t a_base = base;
  const uint32_t b_base = base + STAGES * Cfg::A_BYTES;
  const uint32_t s_base = base + STAGES * Cfg::STAGE_BYTES;  // state ring
  uint8_t* s_gen = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + NBUF * Cfg::BUF_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);
  auto bar = [&](int i) { return ptx::smem_u32(bars + i); };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(STAGES + s); };
  auto tfull_bar = [&](int b) { return bar(2 * STAGES + b); };
  auto tempty_bar = [&](int b) { return bar(2 * STAGES + 2 + b); };
  auto sfull_bar = [&](int b) { return bar(2 * STAGES + 4 + b); };
  auto sempty_bar = [&](int b) { return bar(2 * STAGES + 4 + NBUF + b); };
  auto sdone_bar = [&](int b) { return bar(2 * STAGES + 4 + 2 * NBUF + b); };

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
    for (int b = 0; b < NBUF; ++b) {
      ptx::mbar_init(sfull_bar(b), 1);
      ptx::mbar_init(sempty_bar(b), 1);
      ptx::mbar_init(sdone_bar(b), 8);
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
  const int KB = args.npad / Cfg::BK;
  constexpr int CHUNKS = BN / CW;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------- operand producer
      ptx::prefetch_tmap(&maps.J);
      ptx::prefetch_tmap(&maps.Gin);
      int stage = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m_blk = t % args.num_m;
        const int n_blk = t / args.num_m;
        for (int kb = 0; kb < KB; ++kb) {
          ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
          ptx::mbar_arrive_expect_tx(full_bar(stage), Cfg::STAGE_BYTES);
          ptx::tma_load_2d(a_base + stage * Cfg::A_BYTES, &maps.J, full_bar(stage), kb * Cfg::BK, m_blk * Cfg::BM);
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl)
            ptx::tma_load_2d(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES, &maps.Gin, full_bar(stage),
                             kb * Cfg::BK, pl * args.rpad + n_blk * BN);
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      constexpr uint32_t idesc_s = ptx::idesc_i8(128, BN, true, true);
      constexpr uint32_t idesc_u = ptx::idesc_i8(128, BN, true, false);
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        const int buf = lt & 1;
        ptx::mbar_wait(tempty_bar(buf), ((lt >> 1) & 1) ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_base = tmem_base + buf * Cfg::ACC_COLS;
        for (int kb = 0; kb < KB; ++kb) {
          ptx::mbar_wait(full_bar(stage), ph);
          ptx::tc_fence_after();
          const uint64_t adesc = ptx::smem_desc_k_sw128(a_base + stage * Cfg::A_BYTES);
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl) {
            const uint64_t bdesc = ptx::smem_desc_k_sw128(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES);
            const uint32_t idesc = (NPLANES == 1 || pl == NPLANES - 1) ? idesc_s : idesc_u;
#pragma unroll
            for (int k = 0; k < Cfg::BK / 32; ++k)
              ptx::mma_i8(d_base + pl * BN, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
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
  } else if (warp == 2) {
    if (lane == 0) {  // ----------------------------------------- state loader
      ptx::prefetch_tmap(&maps.X);
      ptx::prefetch_tmap(&maps.Y);
      ptx::prefetch_tmap(&maps.P);
      int ck = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int i0 = (t % args.num_m) * Cfg::BM;
        const int rb = (t / args.num_m) * BN;
        for (int c = 0; c < CHUNKS; ++c, ++ck) {
          const int b = ck % NBUF;
          ptx::mbar_wait(sempty_bar(b), ((ck / NBUF) & 1) ^ 1u);
          ptx::mbar_arrive_expect_tx(sfull_bar(b), 3 * Cfg::ST_ARR);
          const uint32_t sb = s_base + b * Cfg::BUF_BYTES;
          ptx::tma_load_2d(sb, &maps.X, sfull_bar(b), i0, rb + c * CW);
          ptx::tma_load_2d(sb + Cfg::ST_ARR, &maps.Y, sfull_bar(b), i0, rb + c * CW);
          ptx::tma_load_2d(sb + 2 * Cfg::ST_ARR, &maps.P, sfull_bar(b), i0, rb + c * CW);
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ----------------------------------------- state storer
      ptx::prefetch_tmap(&maps.Gout);
      int ck = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int i0 = (t % args.num_m) * Cfg::BM;
        const int rb = (t / args.num_m) * BN;
        for (int c = 0; c < CHUNKS; ++c, ++ck) {
          const int b = ck % NBUF;
          ptx::mbar_wait(sdone_bar(b), (ck / NBUF) & 1);
          const uint32_t sb = s_base + b * Cfg::BUF_BYTES;
          const int r0 = rb + c * CW;
          ptx::tma_store_2d(&maps.X, sb, i0, r0);
          ptx::tma_store_2d(&maps.Y, sb + Cfg::ST_ARR, i0, r0);
          ptx::tma_store_2d(&maps.P, sb + 2 * Cfg::ST_ARR, i0, r0);
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl)
            ptx::tma_store_2d(&maps.Gout, sb + 3 * Cfg::ST_ARR + pl * Cfg::ST_G, i0,
                              (NPLANES == 1 ? 0 : pl * args.rpad) + r0);
          ptx::bulk_commit();
          ptx::bulk_wait_read0();
          ptx::mbar_arrive(sempty_bar(b));
        }
      }
      ptx::bulk_wait0();
    }
  } else {
    // ------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const int srow = q * 32 + lane;  // spin within the 128-row tile
    PhaseConsts k = args.k;
    const uint64_t m = (args.m_dev ? *args.m_dev : 0ull) + static_cast<uint64_t>(args.m_off);
    k.denom = static_cast<float>(args.M - m);
    int ck = 0;
    int lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      const int buf = lt & 1;
      ptx::mbar_wait(tfull_bar(buf), (lt >> 1) & 1);
      __syncwarp();
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * Cfg::ACC_COLS;
      for (int c = 0; c < CHUNKS; ++c, ++ck) {
        const int b = ck % NBUF;
        const int col0 = c * CW + h * CWH;  // accumulator column of this thread's first replica
        float F[CWH];
        if (NPLANES == 1) {
          uint32_t v[CWH];
          ptx::tmem_ld<CWH>(t_row + col0, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < CWH; ++j) F[j] = static_cast<float>(static_cast<int32_t>(v[j]));
        } else {
          long long tot[CWH];
#pragma unroll
          for (int j = 0; j < CWH; ++j) tot[j] = 0;
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl) {
            uint32_t v[CWH];
            ptx::tmem_ld<CWH>(t_row + pl * BN + col0, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CWH; ++j) tot[j] += static_cast<long long>(static_cast<int32_t>(v[j])) << (8 * pl);
          }
#pragma unroll
          for (int j = 0; j < CWH; ++j) F[j] = __fmul_rn(__ll2float_rn(tot[j]), 0x1p-30f);
        }
        ptx::mbar_wait(sfull_bar(b), (ck / NBUF) & 1);
        float* xs = reinterpret_cast<float*>(s_gen + b * Cfg::BUF_BYTES);
        float* ys = xs + CW * Cfg::BM;
        float* ps = ys + CW * Cfg::BM;
        uint8_t* gs = reinterpret_cast<uint8_t*>(ps + CW * Cfg::BM);
#pragma unroll
        for (int j = 0; j < CWH; ++j) {
          const int idx = (h * CWH + j) * Cfg::BM + srow;
          float xv = xs[idx], yv = ys[idx], pv = ps[idx];
          gsb_phase(F[j], xv, yv, pv, k);
          xs[idx] = xv;
          ys[idx] = yv;
          ps[idx] = pv;
          if (NPLANES == 1) {
            gs[idx] = static_cast<uint8_t>(sgn8(xv));
          } else {
            const uint32_t qv = static_cast<uint32_t>(quant30(xv));
#pragma unroll
            for (int pl = 0; pl < NPLANES; ++pl) gs[pl * Cfg::ST_G + idx] = static_cast<uint8_t>(qv >> (8 * pl));
          }
        }
        ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA store
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(sdone_bar(b));
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
