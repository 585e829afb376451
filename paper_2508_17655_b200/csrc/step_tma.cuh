// The hot path: many GSB time steps of every replica in ONE persistent launch.
//
// Semantics per step: sbopt::step (/root/reference/proj/core/src/engine.cpp:55-110)
// for all R replicas,
//
//   F[i, r] = sum_j J[i, j] * G_t[r, j]         tcgen05.mma kind::i8 -> s32 in TMEM
//   (x, y, p)[r, i] <- phase(F[i, r])           fused epilogue (gsb_phase.cuh)
//   G_{t+1}[r, i] <- sgn(x) | fixed-point planes
//
// Work decomposition. A tile is (step t, replica block n of BN replicas, spin
// block m of 128 spins); tiles are numbered g = s*T + n*num_m + m (s = t - t_begin,
// T = num_m*num_n) and dealt round-robin to the persistent CTAs (one per SM),
// each of which walks its tiles in increasing g. Step t+1 of replica block n
// needs every spin of G_{t+1}[n] and of (x, y, p)[n], i.e. the num_m tiles
// (t, n, *): a per-block completion counter done[n] (released by the storer
// once a tile's TMA stores have completed, acquired by the operand producer and
// the state loader before they touch block n of step t+1) replaces the global
// step barrier. Replica blocks are independent, so the pipeline never drains
// between steps and there is no per-step launch; the dependency always points
// to smaller tile ids, so with all CTAs co-resident the schedule cannot
// deadlock. The WAR hazard on the ping-pong B buffers is covered by the same
// counter: G_{t+2} overwrites G_t only after all readers of G_t[n] (the MMAs of
// tiles (t, n, *)) have completed.
//
// Inside a CTA (640 threads):
//   warp 0  TMA producer: J (A, 128x128 B) and G_t (B, BN x 128 B) K-stages, 128B swizzle
//   warp 1  MMA issuer (one lane): 4 x tcgen05.mma per K-stage into one of two TMEM
//           accumulators (the epilogue of tile k overlaps the MMA of tile k+1)
//   warp 2  TMEM allocator, then state loader: TMA loads of x, y, p chunks
//           (128 spins x CW replicas) into an NBUF-deep shared-memory ring
//   warp 3  state storer: TMA stores of x, y, p and G_{t+1} from the ring; releases done[n]
//   warps 4..19  epilogue: tcgen05.ld of F, phase update in shared memory
// Tensor-map bounds (n spins x R replicas) zero-fill loads and clip stores at
// the edges; HBM traffic is exactly 12 B read + 12 B written per spin-update
// plus the 1 (sign) or 4 (planes) bytes of G_{t+1}.
#pragma once

#include <cstdint>
#include <cuda.h>

#include "gsb_phase.cuh"
#include "ptx.cuh"

#ifndef SBG_FX_BK
#define SBG_FX_BK 128
#endif

namespace sbg {

template <int NPLANES, int BN, int STAGES_, int NBUF_, int NA_ = 1>
struct TmaStepCfg {
  static constexpr int BM = 128;
  static constexpr int NA = NA_;                        // J byte planes (1: int8 J; 3: fixed-point real J)
  // K bytes per operand stage: 128 (128-byte swizzle). SBG_FX_BK=64 (dev): real J x 4 digit
  // planes in 64-byte stages (64-byte swizzle), twice as many at half the size -- bitwise
  // equal, measured slower at C4 (257 vs 244 us/step)
  static constexpr int BK = (NA_ > 1 && NPLANES == 4) ? SBG_FX_BK : 128;
  static constexpr int NW = NA + NPLANES - 1;           // distinct plane weights 2^(8(a+b))
  // fixed-point real J with continuous x: the products of weight w = a + b < W0 (J's two low
  // bytes times q's two low digits: < 2^-27 of the field, below its fp32 rounding) are not
  // formed: 9 of the 12 plane products; accumulator k holds weight W0 + k
  static constexpr int W0 = (NA > 1 && NPLANES == 4) ? 2 : 0;
  static constexpr int A_BYTES = BM * BK;               // one J plane tile
  static constexpr int B_PLANE_BYTES = BN * BK;
  static constexpr int STAGE_BYTES = NA * A_BYTES + NPLANES * B_PLANE_BYTES;
  static constexpr int STAGES = STAGES_;                // operand ring depth
  static constexpr int EPI_WARPS = 16;                  // 4 per TMEM lane quadrant
  static constexpr int CW = 16;                         // replicas per state chunk
  static constexpr int CWQ = CW / (EPI_WARPS / 4);      // replicas per epilogue thread per chunk
  static constexpr int NBUF = NBUF_;                    // state ring depth
  static constexpr int ST_ARR = CW * BM * 4;            // one fp32 array chunk: 8 KB
  static constexpr int ST_G = CW * BM;                  // one byte plane chunk: 2 KB
  static constexpr int BUF_RAW = 3 * ST_ARR + NPLANES * ST_G;
  static constexpr int BUF_BYTES = (BUF_RAW + 1023) / 1024 * 1024;
  static constexpr int ACC_COLS = (NW - W0) * BN;       // one accumulator per formed plane weight
  // accumulator buffers: 2 when they fit TMEM, else 1 (the epilogue then drains all of a
  // tile's accumulator columns first and releases them before its state chunks)
  static constexpr int ABUF = 2 * ACC_COLS <= 512 ? 2 : 1;
  // one MMA per J plane over all (signed digit) planes of B (N = NPLANES * BN <= 256)
  static constexpr bool MERGED = NPLANES > 1 && NPLANES * BN <= 256;
  static constexpr int TMEM_COLS = ABUF * ACC_COLS <= 256 ? 256 : 512;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int NUM_BARS = 2 * STAGES + 4 + 3 * NBUF;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + NBUF * BUF_BYTES + 1024 + 8 * NUM_BARS + 64;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(BN % CW == 0, "chunking");
  static_assert(ABUF * ACC_COLS <= 512, "TMEM allocation");
};

struct TmaMaps {
  CUtensorMap J;        // A operand, int8 [npad][npad], 128B swizzle
  CUtensorMap Gin[2];   // B operand of step parity 0/1: [NPLANES*rpad][npad], 128B swizzle
  CUtensorMap Gout[2];  // next B operand of step parity 0/1 (sign: [R][n]; planes: [NPLANES*rpad][n])
  CUtensorMap X, Y, P;  // fp32 state [R][n] (row pitch ld)
};

struct MultiStepArgs {
  int32_t n, npad, R, rpad;
  int32_t num_m, num_n;
  PhaseConsts k;     // a, c, dt (inv is per tile)
  uint64_t M;        // schedule length
  uint64_t t_begin;  // first step index of this launch
  int32_t nsteps;    // steps in this launch
  uint32_t* done;    // [num_n] tiles completed per replica block, zero at launch
  int32_t dbg;       // dev experiments: 1 = no state traffic, 2 = no MMA, 3 = no MMA and no compute
  int32_t fx_exp;    // NA > 1: F = sum_w acc_w 2^(8w + fx_exp) (fixed-point J scale + x scale)
  // --- row sharding. Unsharded: kpad = npad, num_m_total = num_m,
  // col0 = 0, done_base = 0, npeers = 0.
  int32_t kpad;          // K extent of the contraction (global padded n)
  int32_t num_m_total;   // 128-spin row tiles over all ranks (dependency count per step)
  int32_t col0;          // this rank's first spin (column offset of its slab of G)
  uint32_t done_base;    // done[] value at launch (counters run on across launches)
  int32_t npeers;        // other ranks that receive this rank's G slab
  uint32_t* err;         // row shards: set to 1 when a peer wait times out (the launch then
                         // finishes with garbage instead of hanging; the host reports it)
  int64_t g_ld;          // row pitch (bytes) of the G buffers
  uint8_t* peer_g[2][7]; // peers' G buffers for step parity 0/1 (NVLink peer / IPC pointers)
  uint32_t* peer_done[7];
  const float* a_rep;    // optional per-replica control strength A (sweeps over A in one launch)
  // --- K split (CTA-pair kernel, sign plane): each pair tile's K range runs as ksplit units on
  // different pairs; units 0..ksplit-2 store their partial fields (exact integers) into
  // fpart[kp][rpad][npad] and count kdone[n_blk * num_m + m_blk]; unit ksplit-1 adds them to
  // its own and runs the state update. ksplit <= 1: no split.
  int32_t ksplit;
  int32_t ktail;  // > 0: only the last ktail pair tiles of a step are split (the rest run whole)
  unsigned long long* utrace;  // dev (SBG_PAIR_TRACE): per (CTA, unit slot) %globaltimer stamps, 8 each
  float *sx, *sy, *sp;         // replica-major state [rpad][npad] (pair kernel with direct state access)
  float* fpart;
  uint32_t* kdone;
  // CTA-pair kernel tile order within a step: 0 = spin pair-blocks fastest, 1 = replica blocks
  // fastest (the replica blocks of one pair-block run side by side and share its J reads in L2)
  int32_t n_fast;
  // Fused rank emulation (CTA-pair kernel instantiated with FUSED, test-only): `ranks` row
  // shards of ONE GPU in one cooperative launch, CTAs [r * grid / ranks, (r + 1) * grid / ranks)
  // running rank r with rank_args[r] / rank_maps[r] (device memory), so the multi-step
  // cross-rank waits execute inside one launch (kernels that wait on one another must never be
  // separate launches on one GPU).
  int32_t ranks;
  const MultiStepArgs* rank_args;
  const TmaMaps* rank_maps;
};
constexpr int MAX_PEERS = 7;

namespace dep {
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Block until `need` tiles of replica block n are complete, then order the
// caller's subsequent async-proxy (TMA) reads after that observation.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
#ifndef SBG_POLL
#define SBG_POLL 0  // 0: ld.acquire + 32 ns sleep per poll; 1: relaxed spin, then one acquire; 2: acquire spin
#endif
__device__ __forceinline__ void wait_block(const uint32_t* done, int n, uint32_t base, uint32_t need) {
  if (need == 0) return;
#if SBG_POLL == 1
  while (ld_relaxed(done + n) - base < need) {
  }
  (void)ld_acquire(done + n);
#elif SBG_POLL == 2
  while (ld_acquire(done + n) - base < need) {
  }
#else
  while (ld_acquire(done + n) - base < need) __nanosleep(32);
#endif
  fence_proxy_async_global();
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void release_add_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Sharded variant: counters are incremented by peer GPUs over NVLink (sys scope) and run on
// across launches (base = the count every rank's previous launches reach). No need == 0
// shortcut: step 0 of a later launch must still see every peer's final step of the previous
// one (done >= base), so that it neither reads a stale slab nor overwrites a G buffer a slower
// peer is still reading. Signed, wrap-safe compare.
// A wait longer than SHARD_WAIT_NS (a peer rank died or was never launched) sets *err and
// gives up; every other waiter then gives up at once.
constexpr uint64_t SHARD_WAIT_NS = 4000000000ull;
__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wait_block_sys(const uint32_t* done, int n, uint32_t base, uint32_t need,
                                               uint32_t* err) {
  const uint32_t target = base + need;
  if (static_cast<int32_t>(ld_acquire_sys(done + n) - target) < 0) {
    const uint64_t t0 = now_ns();
    while (static_cast<int32_t>(ld_acquire_sys(done + n) - target) < 0) {
      __nanosleep(64);
      if (err && (*reinterpret_cast<volatile uint32_t*>(err) != 0 || now_ns() - t0 > SHARD_WAIT_NS)) {
        atomicExch(err, 1u);
        break;
      }
    }
  }
  fence_proxy_async_global();
}
}  // namespace dep

template <int NPLANES, int BN, int STAGES_, int NBUF_, int NA_ = 1>
__global__ void __launch_bounds__(TmaStepCfg<NPLANES, BN, STAGES_, NBUF_, NA_>::THREADS, 1)
    gsb_multistep_kernel(const __grid_constant__ TmaMaps maps, const MultiStepArgs args) {
  using Cfg = TmaStepCfg<NPLANES, BN, STAGES_, NBUF_, NA_>;
  constexpr int NA = Cfg::NA;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int NBUF = Cfg::NBUF;
  constexpr int CW = Cfg::CW;
  constexpr int CWQ = Cfg::CWQ;
  constexpr int CHUNKS = BN / CW;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_addr);
  const uint32_t a_base = base;                                // J plane tiles [STAGES][NA]
  const uint32_t b_base = base + STAGES * NA * Cfg::A_BYTES;   // B plane tiles [STAGES][NPLANES]
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
      ptx::mbar_init(tempty_bar(b), Cfg::EPI_WARPS);
    }
    for (int b = 0; b < NBUF; ++b) {
      ptx::mbar_init(sfull_bar(b), 1);
      ptx::mbar_init(sempty_bar(b), 1);
      ptx::mbar_init(sdone_bar(b), Cfg::EPI_WARPS);
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

  const int T = args.num_m * args.num_n;
  const int total = T * args.nsteps;
  const int KB = args.kpad / Cfg::BK;
  const bool sharded = args.npeers > 0;
  auto wait_dep = [&](int n_blk, int s) {
    const uint32_t need = static_cast<uint32_t>(s * args.num_m_total);
    if (sharded)
      dep::wait_block_sys(args.done, n_blk, args.done_base, need, args.err);
    else
      dep::wait_block(args.done, n_blk, args.done_base, need);
  };

  if (warp == 0) {
    if (SBG_DBG(args) < 2) {  // ------------------------------------------ operand producer
      // whole warp walks the schedule (uniform values), one elected lane issues TMA
      if (ptx::elect_one()) {
        ptx::prefetch_tmap(&maps.J);
        ptx::prefetch_tmap(&maps.Gin[0]);
        ptx::prefetch_tmap(&maps.Gin[1]);
      }
      int stage = 0;
      uint32_t ph = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int s = g / T, w = g % T;
        const int n_blk = w / args.num_m, m_blk = w % args.num_m;
        wait_dep(n_blk, s);
        const CUtensorMap* gin = &maps.Gin[s & 1];
        for (int kb = 0; kb < KB; ++kb) {
          ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
          if (ptx::elect_one()) {
            ptx::mbar_arrive_expect_tx(full_bar(stage), Cfg::STAGE_BYTES);
#pragma unroll
            for (int ap = 0; ap < NA; ++ap)
              ptx::tma_load_2d(a_base + (stage * NA + ap) * Cfg::A_BYTES, &maps.J, full_bar(stage), kb * Cfg::BK,
                               ap * args.num_m * Cfg::BM + m_blk * Cfg::BM);
#pragma unroll
            for (int pl = 0; pl < NPLANES; ++pl)
              ptx::tma_load_2d(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES, gin, full_bar(stage),
                               kb * Cfg::BK, pl * args.rpad + n_blk * BN);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (SBG_DBG(args) < 2) {  // ------------------------------------------------ MMA issuer
      // the whole warp walks the (warp-uniform) schedule; one elected lane issues
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x, ++lt) {
        const int buf = lt % Cfg::ABUF;
        ptx::mbar_wait(tempty_bar(buf), ((lt / Cfg::ABUF) & 1) ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_base = tmem_base + buf * Cfg::ACC_COLS;
        for (int kb = 0; kb < KB; ++kb) {
          ptx::mbar_wait(full_bar(stage), ph);
          ptx::tc_fence_after();
          const bool issuer = ptx::elect_one();
          if (Cfg::MERGED && issuer) {
            // all NPLANES signed digit planes of B in one MMA per J plane ap: the product
            // J_ap x d_p lands in accumulator ap + p (columns (ap + p) BN ..), as below. In a
            // tile's first K-chunk, plane NPLANES-1 of ap >= 1 opens accumulator ap + NPLANES-1
            // (a separate N = BN MMA without accumulate); everything else accumulates.
            // With W0 > 0, J plane ap multiplies digit planes pl0 = max(0, W0 - ap) .. NPLANES-1
            // only (a contiguous run of B rows: N = (NPLANES - pl0) BN) into accumulators
            // ap + pl0 - W0 ..; ap = 0 opens accumulators 0 .. NPLANES-1-W0.
            constexpr uint32_t NB = BN;
#pragma unroll
            for (int k = 0; k < Cfg::BK / 32; ++k) {
#pragma unroll
              for (int ap = 0; ap < NA; ++ap) {
                const int pl0 = Cfg::W0 - ap > 0 ? Cfg::W0 - ap : 0;
                const uint32_t np = static_cast<uint32_t>(NPLANES - pl0);
                const bool a_signed = NA == 1 || ap == NA - 1;
                const uint64_t adesc = ptx::smem_desc_k<Cfg::BK>(a_base + (stage * NA + ap) * Cfg::A_BYTES) + 2 * k;
                const uint64_t bd0 =
                    ptx::smem_desc_k<Cfg::BK>(b_base + (stage * NPLANES + pl0) * Cfg::B_PLANE_BYTES) + 2 * k;
                const uint32_t d = d_base + (ap + pl0 - Cfg::W0) * NB;
                if (kb == 0 && k == 0 && ap > 0) {
                  const uint64_t bdl =
                      ptx::smem_desc_k<Cfg::BK>(b_base + (stage * NPLANES + NPLANES - 1) * Cfg::B_PLANE_BYTES);
                  if (np > 1)
                    ptx::mma_i8(d, adesc, bd0, ptx::idesc_i8(128, (np - 1) * NB, a_signed, true), true);
                  ptx::mma_i8(d + (np - 1) * NB, adesc, bdl, ptx::idesc_i8(128, NB, a_signed, true), false);
                } else {
                  ptx::mma_i8(d, adesc, bd0, ptx::idesc_i8(128, np * NB, a_signed, true), (kb | k | ap) != 0);
                }
              }
            }
            ptx::mma_commit(empty_bar(stage));
          } else if (!Cfg::MERGED && issuer) {
#pragma unroll
            for (int ap = 0; ap < NA; ++ap) {
              const uint64_t adesc = ptx::smem_desc_k<Cfg::BK>(a_base + (stage * NA + ap) * Cfg::A_BYTES);
#pragma unroll
              for (int pl = 0; pl < NPLANES; ++pl) {
                const uint64_t bdesc = ptx::smem_desc_k<Cfg::BK>(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES);
                // J planes: only the top plane is signed; B: sign plane or signed digit planes
                const uint32_t idesc = ptx::idesc_i8(128, BN, NA == 1 || ap == NA - 1, true);
                // products of equal weight 2^(8(ap+pl)) share one accumulator; the first
                // pair of each weight (in this loop order) starts it at kb == 0
                const int w = ap + pl;
                if (w < Cfg::W0) continue;  // product not formed (see W0)
                const bool first_pair = ap == (w - (NPLANES - 1) > 0 ? w - (NPLANES - 1) : 0);
#pragma unroll
                for (int k = 0; k < Cfg::BK / 32; ++k)
                  ptx::mma_i8(d_base + (w - Cfg::W0) * BN, adesc + 2 * k, bdesc + 2 * k, idesc,
                              (kb | k) != 0 || !first_pair);
              }
            }
            ptx::mma_commit(empty_bar(stage));
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
        if (ptx::elect_one()) ptx::mma_commit(tfull_bar(buf));
        __syncwarp();
      }
    }
  } else if (warp == 2) {
    if (lane == 0 && SBG_DBG(args) != 1) {  // ------------------------------- state loader
      ptx::prefetch_tmap(&maps.X);
      ptx::prefetch_tmap(&maps.Y);
      ptx::prefetch_tmap(&maps.P);
      int ck = 0;
      for (int g = blockIdx.x; g < total; g += gridDim.x) {
        const int s = g / T, w = g % T;
        const int n_blk = w / args.num_m, m_blk = w % args.num_m;
        wait_dep(n_blk, s);
        const int i0 = m_blk * Cfg::BM, rb = n_blk * BN;
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
    // ------------------------------------------------------------------ state storer
    // lane 0 drives the TMA stores; in sharded runs the whole warp also pushes the
    // freshly computed slab of G_{t+1} into every peer's buffer (NVLink stores) so
    // the next step's contraction on every rank sees all spins.
    if (lane == 0) {
      ptx::prefetch_tmap(&maps.Gout[0]);
      ptx::prefetch_tmap(&maps.Gout[1]);
    }
    int ck = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x) {
      const int s = g / T, w = g % T;
      const int n_blk = w / args.num_m, m_blk = w % args.num_m;
      const int i0 = m_blk * Cfg::BM, rb = n_blk * BN;
      const CUtensorMap* gout = &maps.Gout[s & 1];
      for (int c = 0; c < CHUNKS; ++c, ++ck) {
        const int b = ck % NBUF;
        ptx::mbar_wait(sdone_bar(b), (ck / NBUF) & 1);
        const uint32_t sb = s_base + b * Cfg::BUF_BYTES;
        const int r0 = rb + c * CW;
        if (lane == 0) {
          if (SBG_DBG(args) != 1) {
            ptx::tma_store_2d(&maps.X, sb, i0, r0);
            ptx::tma_store_2d(&maps.Y, sb + Cfg::ST_ARR, i0, r0);
            ptx::tma_store_2d(&maps.P, sb + 2 * Cfg::ST_ARR, i0, r0);
#pragma unroll
            for (int pl = 0; pl < NPLANES; ++pl)
              ptx::tma_store_2d(gout, sb + 3 * Cfg::ST_ARR + pl * Cfg::ST_G, args.col0 + i0,
                                (NPLANES == 1 ? 0 : pl * args.rpad) + r0);
          }
          ptx::bulk_commit();
        }
        if (sharded) {
          // chunk of G: CW replica rows x 128 spins (128 contiguous bytes each), per plane
          const uint8_t* gs = s_gen + b * Cfg::BUF_BYTES + 3 * Cfg::ST_ARR;
          for (int pr = 0; pr < args.npeers; ++pr) {
            uint8_t* dst0 = args.peer_g[s & 1][pr];
#pragma unroll
            for (int pl = 0; pl < NPLANES; ++pl) {
              for (int e = lane; e < CW * Cfg::BM / 16; e += 32) {  // 16-byte pieces
                const int row = e / (Cfg::BM / 16), piece = e % (Cfg::BM / 16);
                const int rr = r0 + row;
                if (rr >= args.R) continue;
                const int spin = args.col0 + i0 + piece * 16;
                const uint4 v = *reinterpret_cast<const uint4*>(gs + pl * Cfg::ST_G + row * Cfg::BM + piece * 16);
                *reinterpret_cast<uint4*>(dst0 + (static_cast<size_t>(NPLANES == 1 ? 0 : pl * args.rpad) + rr) *
                                                     args.g_ld + spin) = v;
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          ptx::bulk_wait_read0();  // smem slot reusable as soon as the engine has read it
          ptx::mbar_arrive(sempty_bar(b));
        }
        __syncwarp();
      }
      // Tile complete: its global writes must land before block n is released.
      // (Deferring this past the next tile's stores deadlocks: the next tile
      // may itself wait on this release.)
      if (lane == 0) {
        ptx::bulk_wait0();
        dep::fence_proxy_async_global();
        if (sharded) {
          __threadfence_system();
          dep::release_add_sys(args.done + n_blk, 1u);
          for (int pr = 0; pr < args.npeers; ++pr) dep::release_add_sys(args.peer_done[pr] + n_blk, 1u);
        } else {
          __threadfence();
          dep::release_add(args.done + n_blk, 1u);
        }
      }
      __syncwarp();
    }
  } else {
    // --------------------------------------------------------------------- epilogue
    const int q = warp & 3;           // TMEM lane quadrant
    const int h = (warp - 4) >> 2;    // column quarter of each chunk
    const int srow = q * 32 + lane;   // spin within the 128-row tile
    PhaseConsts k = args.k;
    int ck = 0;
    int lt = 0;
    for (int g = blockIdx.x; g < total; g += gridDim.x, ++lt) {
      const int s = g / T;
      const int rbase = ((g % T) / args.num_m) * BN;  // first replica of this tile
      k.inv = __frcp_rn(static_cast<float>(args.M - (args.t_begin + static_cast<uint64_t>(s))));
      const int buf = lt % Cfg::ABUF;
      if (SBG_DBG(args) < 2) ptx::mbar_wait(tfull_bar(buf), (lt / Cfg::ABUF) & 1);
      __syncwarp();
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * Cfg::ACC_COLS;
      // the field of chunk c (this thread's CWQ replicas) from the accumulator columns
      auto load_F = [&](int c, float* F) {
        const int col0 = c * CW + h * CWQ;
        if (NA > 1) {
          // fixed-point real J: F = fl32(sum_w fl64(acc_w * 2^(8w + fx_exp))), fixed order
          double f[CWQ];
#pragma unroll
          for (int j = 0; j < CWQ; ++j) f[j] = 0.0;
#pragma unroll
          for (int w = Cfg::W0; w < Cfg::NW; ++w) {
            uint32_t v[CWQ];
            ptx::tmem_ld<CWQ>(t_row + (w - Cfg::W0) * BN + col0, v);
            ptx::tmem_ld_wait();
            const double sc = ldexp(1.0, 8 * w + args.fx_exp);
#pragma unroll
            for (int j = 0; j < CWQ; ++j)
              f[j] = __dadd_rn(f[j], __dmul_rn(static_cast<double>(static_cast<int32_t>(v[j])), sc));
          }
#pragma unroll
          for (int j = 0; j < CWQ; ++j) F[j] = __double2float_rn(f[j]);
        } else if (NPLANES == 1) {
          uint32_t v[CWQ];
          ptx::tmem_ld<CWQ>(t_row + col0, v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < CWQ; ++j) F[j] = static_cast<float>(static_cast<int32_t>(v[j]));
        } else {
          long long tot[CWQ];
#pragma unroll
          for (int j = 0; j < CWQ; ++j) tot[j] = 0;
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl) {
            uint32_t v[CWQ];
            ptx::tmem_ld<CWQ>(t_row + pl * BN + col0, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CWQ; ++j) tot[j] += static_cast<long long>(static_cast<int32_t>(v[j])) << (8 * pl);
          }
#pragma unroll
          for (int j = 0; j < CWQ; ++j) F[j] = __fmul_rn(__ll2float_rn(tot[j]), 0x1p-30f);
        }
      };
      float Fall[Cfg::ABUF == 1 ? CHUNKS : 1][CWQ];
      if constexpr (Cfg::ABUF == 1) {  // single accumulator buffer: drain it, release it, then update
#pragma unroll
        for (int c = 0; c < CHUNKS; ++c) load_F(c, Fall[c]);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty_bar(buf));
      }
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c, ++ck) {
        const int b = ck % NBUF;
        const int col0 = c * CW + h * CWQ;
        float F[CWQ];
        if constexpr (Cfg::ABUF == 1) {
#pragma unroll
          for (int j = 0; j < CWQ; ++j) F[j] = Fall[c][j];
        } else {
          load_F(c, F);
        }
        if (SBG_DBG(args) != 1) {
          ptx::mbar_wait(sfull_bar(b), (ck / NBUF) & 1);
          float* xs = reinterpret_cast<float*>(s_gen + b * Cfg::BUF_BYTES);
          float* ys = xs + CW * Cfg::BM;
          float* ps = ys + CW * Cfg::BM;
          uint8_t* gs = reinterpret_cast<uint8_t*>(ps + CW * Cfg::BM);
          if (SBG_DBG(args) != 3) {
#pragma unroll
            for (int j = 0; j < CWQ; ++j) {
              const int idx = (h * CWQ + j) * Cfg::BM + srow;
              float xv = xs[idx], yv = ys[idx], pv = ps[idx];
              PhaseConsts kj = k;
              if (args.a_rep) kj.a = args.a_rep[min(rbase + col0 + j, args.R - 1)];
              gsb_phase(F[j], xv, yv, pv, kj);
              xs[idx] = xv;
              ys[idx] = yv;
              ps[idx] = pv;
              if (NPLANES == 1) {
                gs[idx] = static_cast<uint8_t>(sgn8(xv));
              } else {
                const uint32_t qv = qdigits(quant30(xv));
#pragma unroll
                for (int pl = 0; pl < NPLANES; ++pl) gs[pl * Cfg::ST_G + idx] = static_cast<uint8_t>(qv >> (8 * pl));
              }
            }
          }
          ptx::fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the TMA store
        } else {
          float acc = 0.f;
#pragma unroll
          for (int j = 0; j < CWQ; ++j) acc += F[j];
          if (acc == 12345.f) args.done[0] = 0;  // keep the TMEM loads alive
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(sdone_bar(b));
      }
      if constexpr (Cfg::ABUF == 2) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(tempty_bar(buf));
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
}

}  // namespace sbg
