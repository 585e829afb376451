// The hot path on CTA pairs: the multi-step dataflow kernel of step_tma.cuh
// with the field contraction issued as tcgen05.mma.cta_group::2 (M = 256 spins
// across the two SMs of a cluster).
//
// Why pairs: per step every replica block re-reads J and every spin block
// re-reads G, so operand bytes per output element are (1/BN + 1/BM). With a
// pair, each CTA stages only its own 128 rows of J and HALF of the B tile, yet
// its TMEM receives a full 128 x N accumulator: operand bytes per output halve
// compared with one CTA, which frees the shared memory the state stream needs
// (a deeper x/y/p ring), and that stream is what bounds the step (SURVEY 8(d):
// 24 B of state per spin-update vs one int8 op pair per J entry).
//
// Protocol (leader = cluster rank 0):
//   full[s]   leader only, count 2: each CTA's producer arrive.expect_tx(own bytes)
//             on the leader's barrier; each CTA's TMA completes tx there (cta_group::2).
//   empty[s]  both CTAs, count 1: the leader's tcgen05.commit multicasts to both.
//   tfull[b]  both CTAs, count 1: multicast commit after the last K-stage of a tile.
//   tempty[b] leader only, count 2*EPI_WARPS: each epilogue warp of both CTAs
//             arrives (the peer's remotely) when its TMEM reads are done.
//   state ring barriers and done[] counters: per CTA, exactly as step_tma.cuh.
// Tile = (step s, replica block n of N_PAIR, spin pair-block mp of 256); CTA rank
// cr owns spins (2 mp + cr)*128 .. +127 and stages B rows n*N_PAIR + cr*N_PAIR/2.
#pragma once

#include <cstdint>
#include <cuda.h>

#include "gsb_phase.cuh"
#include "ptx.cuh"
#include "step_tma.cuh"

#ifndef SBG_PAIR_DIRECT
#define SBG_PAIR_DIRECT 0  // 1: direct-state epilogue (bitwise equal; measured slower: C1 15.8 -> 16.2, C4 199 -> 202 us)
#endif
#ifndef SBG_Q4_EARLY
#define SBG_Q4_EARLY 1  // e2m1 pair kernel drains its single accumulator early (C5 1013 -> 973 us; 0: off)
#endif
#ifndef SBG_PAIR_STATE_PF
#define SBG_PAIR_STATE_PF 0  // 1: L2 prefetch of a tile's state at its start (measured slower at C5: 1043 vs 1014 us)
#endif

namespace sbg {

__device__ __forceinline__ unsigned long long gtimer_pair() {  // dev traces (%globaltimer, ns)
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Q4_ (sign plane only): packed e2m1 J and G with kind::mxf4 MMAs, as in step_resident.cuh
// -- half the J bytes per step (the bound of the J-streaming regime, C5) at twice the MMA
// rate. Its unit scale factors take 16 TMEM columns, so the accumulator is single-buffered
// (N_PAIR = 256 leaves no room for two).
// NA_ = 3 (real J, continuous variants): J as the three fixed-point byte planes of step_tma.cuh
// (u8, u8, s8) times the four signed digit planes of q, the nine products of weight
// 2^(8w), w = a + b >= W0 = 2, one MMA each (N = N_PAIR), into four accumulators; the pair
// halves the shared-memory operand traffic per MMA of the single-CTA real-J kernel, which is
// what bounds that one (C4).
template <int NPLANES, int N_PAIR, int STAGES_, int NBUF_, int CW_ = 16, bool Q4_ = false, int NA_ = 1>
struct PairStepCfg {
  static constexpr bool Q4 = Q4_;
  static constexpr int NA = NA_;                        // J byte planes
  static constexpr int NW = NA + NPLANES - 1;           // distinct plane weights
  static constexpr int W0 = NA > 1 ? 2 : 0;             // products of weight < W0 not formed
  static constexpr int KPB = Q4 ? 2 : 1;                // K elements per operand byte
  static constexpr int BM = 128;                        // spins per CTA
  static constexpr int BK = 128;                        // K bytes per stage
  static constexpr int B_HALF = N_PAIR / 2;             // B rows staged per CTA (per plane)
  static constexpr int A_PLANE_BYTES = BM * BK;         // one J plane tile
  static constexpr int A_BYTES = NA * A_PLANE_BYTES;
  static constexpr int B_PLANE_BYTES = B_HALF * BK;
  static constexpr int STAGE_BYTES = A_BYTES + NPLANES * B_PLANE_BYTES;
  static constexpr int STAGES = STAGES_;
  static constexpr int EPI_WARPS = 16;
  static constexpr int CW = CW_;                        // replicas per state chunk (TMA box rows)
  static constexpr int CWQ = CW / (EPI_WARPS / 4);
  static constexpr int NBUF = NBUF_;
  static constexpr int ST_ARR = CW * BM * 4;
  static constexpr int ST_G = CW * BM / KPB;
  static constexpr int BUF_RAW = 3 * ST_ARR + NPLANES * ST_G;
  static constexpr int BUF_BYTES = (BUF_RAW + 1023) / 1024 * 1024;
  static constexpr int ACC_COLS = (NA > 1 ? NW - W0 : NPLANES) * N_PAIR;  // per CTA per accumulator buffer
  // accumulator buffers: 2 when they fit TMEM; 1 for e2m1 (scale factors) or wide tiles, whose
  // epilogue (non-e2m1) then drains all accumulator columns before the state update
  static constexpr int NACC = (Q4 || 2 * ACC_COLS > 512) ? 1 : 2;
  // e2m1 too with SBG_Q4_EARLY: the single accumulator (the scale factors leave no room for a
  // second) is drained to registers and released before the state update, so the next tile's
  // MMAs overlap the update instead of waiting for it
  static constexpr bool EARLY_DRAIN = (!Q4 || SBG_Q4_EARLY) && NACC == 1;
  // continuous variants (digit planes): x, y, p go between HBM and the epilogue threads' registers
  // directly (coalesced 128 B per warp and replica) instead of through the shared-memory ring and
  // TMA -- the ring then only stages the G planes. Shared memory is what paces these kernels
  // (TMA writes + MMA operand reads + the state passes); this removes four state passes.
  static constexpr bool DIRECT = SBG_PAIR_DIRECT && NPLANES > 1 && !Q4;
  // all digit planes in one MMA (N = NPLANES * N_PAIR <= 256). The pair's output columns are
  // then [CTA 0's B rows][CTA 1's B rows], each [plane][B_HALF replicas]: plane p of replica
  // r (of the tile) sits at column (r / B_HALF) * NPLANES * B_HALF + p * B_HALF + r % B_HALF
  static constexpr bool MERGED = NA == 1 && !Q4 && NPLANES > 1 && NPLANES * N_PAIR <= 256;
  static constexpr int TMEM_COLS = Q4 ? 512 : NACC * ACC_COLS;
  static constexpr uint32_t COL_SF = 512 - 16;          // Q4: unit E8M0 scale factors
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int NUM_BARS = 2 * STAGES + 4 + 3 * NBUF;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + NBUF * BUF_BYTES + 1024 + 8 * NUM_BARS + 64;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(N_PAIR % 32 == 0 && N_PAIR <= 256 && N_PAIR >= 32, "UMMA N for M=256");
  static_assert(N_PAIR % CW == 0, "chunking");
  static_assert(TMEM_COLS == 256 || TMEM_COLS == 512, "TMEM allocation");
  static_assert(!Q4 || (NPLANES == 1 && ACC_COLS <= 496), "e2m1: sign plane, room for the scale factors");
  static_assert(NA == 1 || (NA == 3 && NPLANES == 4 && !Q4), "real J: continuous variants, int8 planes");
};

template <int NPLANES, int N_PAIR, int STAGES_, int NBUF_, int CW_ = 16, bool Q4_ = false, int NA_ = 1,
          bool FUSED = false>
__global__ void __cluster_dims__(2, 1, 1)
    __launch_bounds__(PairStepCfg<NPLANES, N_PAIR, STAGES_, NBUF_, CW_, Q4_, NA_>::THREADS, 1)
        gsb_multistep_pair_kernel(const __grid_constant__ TmaMaps maps_p, const __grid_constant__ MultiStepArgs args_p) {
  using Cfg = PairStepCfg<NPLANES, N_PAIR, STAGES_, NBUF_, CW_, Q4_, NA_>;
  // FUSED: this CTA's rank of a fused row-shard emulation (MultiStepArgs::ranks); rank groups
  // hold an even number of CTAs, so a cluster never straddles two ranks
  const int cpr = FUSED ? static_cast<int>(gridDim.x) / args_p.ranks : static_cast<int>(gridDim.x);
  const int rank = FUSED ? static_cast<int>(blockIdx.x) / cpr : 0;
  const MultiStepArgs& args = FUSED ? args_p.rank_args[rank] : args_p;
  const TmaMaps& maps = FUSED ? args_p.rank_maps[rank] : maps_p;
  const int bid = FUSED ? static_cast<int>(blockIdx.x) % cpr : static_cast<int>(blockIdx.x);
  constexpr int NA = Cfg::NA;
  constexpr int NACC = Cfg::NACC;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int NBUF = Cfg::NBUF;
  constexpr int CW = Cfg::CW;
  constexpr int CWQ = Cfg::CWQ;
  constexpr int CHUNKS = N_PAIR / CW;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_addr);
  const uint32_t a_base = base;
  const uint32_t b_base = base + STAGES * Cfg::A_BYTES;
  const uint32_t s_base = base + STAGES * Cfg::STAGE_BYTES;
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
  const uint32_t cr = ptx::cluster_ctarank();
  const bool leader = cr == 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), 2);
      ptx::mbar_init(empty_bar(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(tfull_bar(b), 1);
      ptx::mbar_init(tempty_bar(b), 2 * Cfg::EPI_WARPS);
    }
    for (int b = 0; b < NBUF; ++b) {
      ptx::mbar_init(sfull_bar(b), 1);
      ptx::mbar_init(sempty_bar(b), 1);
      ptx::mbar_init(sdone_bar(b), Cfg::EPI_WARPS);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc_pair(ptx::smem_u32(tmem_slot), Cfg::TMEM_COLS);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if constexpr (Cfg::Q4) {  // unit E8M0 scale factors (127 = 2^0) in columns [COL_SF, 512)
    if (warp >= 4 && warp < 8) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
      const uint32_t t = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + Cfg::COL_SF;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t), "r"(v[0]),
                   "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                   : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t + 8), "r"(v[0]),
                   "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                   : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    ptx::tc_fence_after();
  }

  const int num_mp = args.num_m / 2;
  const int T2 = num_mp * args.num_n;  // pair tiles per step
  const int KS = args.ksplit > 1 ? args.ksplit : 1;
  // K split: the last TT pair tiles of each step run as KS K-part units (parts adjacent; all
  // tiles when ktail <= 0), the first T2 - TT as whole units -- with ktail = T2 mod npairs the
  // split fills the last, partial round of tiles instead of leaving pairs idle
  const int TT = KS > 1 ? (args.ktail > 0 ? min(args.ktail, T2) : T2) : 0;
  const int TW = T2 - TT;
  const int T2K = TW + TT * KS;        // work units per step
  // unit g -> step s, pair tile w, K part kp of ks
  auto unit = [&](int g, int& s, int& w, int& kp, int& ks) {
    s = g / T2K;
    const int u = g % T2K;
    if (u < TW) {
      w = u, kp = 0, ks = 1;
    } else {
      w = TW + (u - TW) / KS, kp = (u - TW) % KS, ks = KS;
    }
  };
  auto n_of = [&](int w) { return args.n_fast ? w % args.num_n : w / num_mp; };
  auto mp_of = [&](int w) { return args.n_fast ? w / args.num_n : w % num_mp; };
  const int total = T2K * args.nsteps;
  const int pair = bid >> 1;
  const int npairs = cpr >> 1;
  const int KB = args.kpad / (Cfg::BK * Cfg::KPB);
  // Row shards (npeers > 0, K7): counters also count the peers' m-blocks (num_m_total per
  // step) and are released by other GPUs over NVLink, so waits are system-scope.
  const bool sharded = args.npeers > 0;
  auto wait_dep = [&](int n_blk, int s) {
    const uint32_t need = static_cast<uint32_t>(s * args.num_m_total);
    if (sharded)
      dep::wait_block_sys(args.done, n_blk, args.done_base, need, args.err);
    else
      dep::wait_block(args.done, n_blk, args.done_base, need);
  };

  if (warp == 0) {
    if (SBG_DBG(args) < 2) {  // ------------------------------------------- operand producer (both CTAs)
      // whole warp walks the schedule (uniform values), one elected lane issues TMA
      if (ptx::elect_one()) {
        ptx::prefetch_tmap(&maps.J);
        ptx::prefetch_tmap(&maps.Gin[0]);
        ptx::prefetch_tmap(&maps.Gin[1]);
      }
      int stage = 0;
      uint32_t ph = 0;
      const uint64_t keep = ptx::policy_evict_last();  // J and G are re-read every step: keep them in L2
      for (int g = pair; g < total; g += npairs) {
        int s, w, kp, ks;
        unit(g, s, w, kp, ks);
        const int n_blk = n_of(w), mp = mp_of(w);
        const int m_blk = 2 * mp + static_cast<int>(cr);
        wait_dep(n_blk, s);
        const CUtensorMap* gin = &maps.Gin[s & 1];
        for (int kb = kp * KB / ks; kb < (kp + 1) * KB / ks; ++kb) {
          ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
          if (ptx::elect_one()) {
            const uint32_t fb = ptx::mapa(full_bar(stage), 0);  // the leader's full barrier
            ptx::mbar_arrive_expect_tx_cluster(fb, Cfg::STAGE_BYTES);
#pragma unroll
            for (int ap = 0; ap < NA; ++ap)  // J planes stacked [NA][npad] rows in one map
              ptx::tma_load_2d_pair_hint(a_base + stage * Cfg::A_BYTES + ap * Cfg::A_PLANE_BYTES, &maps.J, fb,
                                         kb * Cfg::BK, ap * args.num_m * Cfg::BM + m_blk * Cfg::BM, keep);
#pragma unroll
            for (int pl = 0; pl < NPLANES; ++pl)
              ptx::tma_load_2d_pair_hint(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES, gin, fb, kb * Cfg::BK,
                                         pl * args.rpad + n_blk * N_PAIR + static_cast<int>(cr) * Cfg::B_HALF, keep);
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
    if (leader && SBG_DBG(args) < 2) {  // --------------------------------- MMA issuer (leader CTA only)
      // whole warp walks the schedule; one elected lane issues (uniform descriptors)
      constexpr uint32_t idesc_s = Cfg::Q4 ? ptx::idesc_mxf4(256, N_PAIR) : ptx::idesc_i8(256, N_PAIR, true, true);
      // MERGED: the NPLANES signed digit planes of B are consecutive smem tiles, i.e. one
      // B operand of NPLANES * N_PAIR rows: one MMA per K-chunk reads A once for all planes
      constexpr uint32_t idesc_m = ptx::idesc_i8(256, Cfg::MERGED ? NPLANES * N_PAIR : N_PAIR, true, true);
      const uint32_t sf = tmem_base + Cfg::COL_SF;
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int g = pair; g < total; g += npairs, ++lt) {
        const int buf = lt % NACC;
        int s_, w_, kp, ks;
        unit(g, s_, w_, kp, ks);
        const int kb0 = kp * KB / ks;
        auto ust = [&](int k) {
          if (SBG_HOOK_PTR(args.utrace) && lt < 64 && lane == 0)
            SBG_HOOK_PTR(args.utrace)[(static_cast<size_t>(blockIdx.x) * 64 + lt) * 8 + k] = gtimer_pair();
        };
        ust(5);
        ptx::mbar_wait(tempty_bar(buf), ((lt / NACC) & 1) ^ 1u);
        ust(0);
        ptx::tc_fence_after();
        const uint32_t d_base = tmem_base + buf * Cfg::ACC_COLS;
        for (int kb = kb0; kb < (kp + 1) * KB / ks; ++kb) {
          ptx::mbar_wait(full_bar(stage), ph);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint64_t adesc = ptx::smem_desc_k_sw128(a_base + stage * Cfg::A_BYTES);
            if constexpr (NA > 1) {
              // real J: product (J plane ap, digit plane pl) of weight w = ap + pl >= W0 into
              // accumulator w - W0; the first product of each weight in this loop order opens it
#pragma unroll
              for (int ap = 0; ap < NA; ++ap) {
                const uint64_t ad = ptx::smem_desc_k_sw128(a_base + stage * Cfg::A_BYTES + ap * Cfg::A_PLANE_BYTES);
                const uint32_t idesc = ptx::idesc_i8(256, N_PAIR, ap == NA - 1, true);
#pragma unroll
                for (int pl = 0; pl < NPLANES; ++pl) {
                  const int w = ap + pl;
                  if (w < Cfg::W0) continue;
                  const bool first_pair = ap == (w - (NPLANES - 1) > 0 ? w - (NPLANES - 1) : 0);
                  const uint64_t bdesc = ptx::smem_desc_k_sw128(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES);
#pragma unroll
                  for (int k = 0; k < Cfg::BK / 32; ++k)
                    ptx::mma_i8_pair(d_base + (w - Cfg::W0) * N_PAIR, ad + 2 * k, bdesc + 2 * k, idesc,
                                     (kb != kb0 || k != 0) || !first_pair);
                }
              }
            } else if constexpr (Cfg::MERGED) {
              const uint64_t bdesc = ptx::smem_desc_k_sw128(b_base + stage * NPLANES * Cfg::B_PLANE_BYTES);
#pragma unroll
              for (int k = 0; k < Cfg::BK / 32; ++k)
                ptx::mma_i8_pair(d_base, adesc + 2 * k, bdesc + 2 * k, idesc_m, (kb != kb0 || k != 0));
            } else {
#pragma unroll
              for (int pl = 0; pl < NPLANES; ++pl) {
                const uint64_t bdesc = ptx::smem_desc_k_sw128(b_base + (stage * NPLANES + pl) * Cfg::B_PLANE_BYTES);
#pragma unroll
                for (int k = 0; k < Cfg::BK / 32; ++k) {  // 32 bytes per MMA (K = 32 int8 / 64 e2m1)
                  if constexpr (Cfg::Q4)
                    ptx::mma_mxf4_pair(d_base, adesc + 2 * k, bdesc + 2 * k, idesc_s, sf, (kb != kb0 || k != 0));
                  else
                    ptx::mma_i8_pair(d_base + pl * N_PAIR, adesc + 2 * k, bdesc + 2 * k, idesc_s, (kb != kb0 || k != 0));
                }
              }
            }
            ptx::mma_commit_pair_mc(empty_bar(stage), 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
        if (ptx::elect_one()) ptx::mma_commit_pair_mc(tfull_bar(buf), 0x3);
        __syncwarp();
        ust(1);
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {  // ------------------------------------------------ state loader
      ptx::prefetch_tmap(&maps.X);
      ptx::prefetch_tmap(&maps.Y);
      ptx::prefetch_tmap(&maps.P);
      int ck = 0;
      const uint64_t stream = ptx::policy_evict_first();  // x, y, p are touched once per step
      for (int g = pair; g < total; g += npairs) {
        int s, w, kp, ks;
        unit(g, s, w, kp, ks);
        if (kp != ks - 1) continue;  // only the last K part updates the state
        const int n_blk = n_of(w), mp = mp_of(w);
        wait_dep(n_blk, s);
        const int i0 = (2 * mp + static_cast<int>(cr)) * Cfg::BM, rb = n_blk * N_PAIR;
#if SBG_PAIR_STATE_PF
        // the whole tile's x, y, p into L2 now, while its MMAs run: the 2-deep ring below then
        // refills from L2 during the epilogue instead of paying an HBM round trip per chunk
        for (int c = NBUF; c < CHUNKS; ++c) {
          ptx::tma_prefetch_2d(&maps.X, i0, rb + c * CW);
          ptx::tma_prefetch_2d(&maps.Y, i0, rb + c * CW);
          ptx::tma_prefetch_2d(&maps.P, i0, rb + c * CW);
        }
#endif
        for (int c = 0; c < CHUNKS; ++c, ++ck) {
          const int b = ck % NBUF;
          ptx::mbar_wait(sempty_bar(b), ((ck / NBUF) & 1) ^ 1u);
          if constexpr (Cfg::DIRECT) {  // only the G staging slot: free -> hand it to the epilogue
            ptx::mbar_arrive(sfull_bar(b));
            continue;
          }
          ptx::mbar_arrive_expect_tx(sfull_bar(b), 3 * Cfg::ST_ARR);
          const uint32_t sb = s_base + b * Cfg::BUF_BYTES;
          ptx::tma_load_2d_hint(sb, &maps.X, sfull_bar(b), i0, rb + c * CW, stream);
          ptx::tma_load_2d_hint(sb + Cfg::ST_ARR, &maps.Y, sfull_bar(b), i0, rb + c * CW, stream);
          ptx::tma_load_2d_hint(sb + 2 * Cfg::ST_ARR, &maps.P, sfull_bar(b), i0, rb + c * CW, stream);
        }
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- state storer
    // lane 0 drives the TMA stores; in sharded runs the whole warp also pushes the
    // chunk's slab of G_{t+1} into every peer's buffer (16-byte NVLink stores).
    if (lane == 0) {
      ptx::prefetch_tmap(&maps.Gout[0]);
      ptx::prefetch_tmap(&maps.Gout[1]);
    }
    int ck = 0;
    const uint64_t stream = ptx::policy_evict_first();
    const uint64_t keep = ptx::policy_evict_last();
    constexpr int GROW = Cfg::BM / Cfg::KPB;  // bytes of one replica row of a G chunk
    for (int g = pair; g < total; g += npairs) {
      int s, w, kp, ks;
      unit(g, s, w, kp, ks);
      if (kp != ks - 1) continue;
      const int n_blk = n_of(w), mp = mp_of(w);
      const int i0 = (2 * mp + static_cast<int>(cr)) * Cfg::BM, rb = n_blk * N_PAIR;
      const CUtensorMap* gout = &maps.Gout[s & 1];
      for (int c = 0; c < CHUNKS; ++c, ++ck) {
        const int b = ck % NBUF;
        ptx::mbar_wait(sdone_bar(b), (ck / NBUF) & 1);
        const uint32_t sb = s_base + b * Cfg::BUF_BYTES;
        const int r0 = rb + c * CW;
        if (lane == 0) {
          if constexpr (!Cfg::DIRECT) {
            ptx::tma_store_2d_hint(&maps.X, sb, i0, r0, stream);
            ptx::tma_store_2d_hint(&maps.Y, sb + Cfg::ST_ARR, i0, r0, stream);
            ptx::tma_store_2d_hint(&maps.P, sb + 2 * Cfg::ST_ARR, i0, r0, stream);
          }
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl)
            ptx::tma_store_2d_hint(gout, sb + 3 * Cfg::ST_ARR + pl * Cfg::ST_G, (args.col0 + i0) / Cfg::KPB,
                                   (NPLANES == 1 ? 0 : pl * args.rpad) + r0, keep);
          ptx::bulk_commit();
        }
        if (sharded) {
          const uint8_t* gs = s_gen + b * Cfg::BUF_BYTES + 3 * Cfg::ST_ARR;
          for (int pr = 0; pr < args.npeers; ++pr) {
            uint8_t* dst0 = args.peer_g[s & 1][pr];
#pragma unroll
            for (int pl = 0; pl < NPLANES; ++pl) {
              for (int e = lane; e < CW * GROW / 16; e += 32) {
                const int row = e / (GROW / 16), piece = e % (GROW / 16);
                const int rr = r0 + row;
                if (rr >= args.R) continue;
                const uint4 v = *reinterpret_cast<const uint4*>(gs + pl * Cfg::ST_G + row * GROW + piece * 16);
                *reinterpret_cast<uint4*>(dst0 + (static_cast<size_t>(NPLANES == 1 ? 0 : pl * args.rpad) + rr) *
                                                     args.g_ld + (args.col0 + i0) / Cfg::KPB + piece * 16) = v;
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          ptx::bulk_wait_read0();
          ptx::mbar_arrive(sempty_bar(b));
        }
        __syncwarp();
      }
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
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const int srow = q * 32 + lane;
    const uint32_t tempty_leader0 = ptx::mapa(tempty_bar(0), 0);
    const uint32_t tempty_leader1 = ptx::mapa(tempty_bar(1), 0);
    PhaseConsts k = args.k;
    int ck = 0;
    int lt = 0;
    for (int g = pair; g < total; g += npairs, ++lt) {
      int s, w, kp, ks;
      unit(g, s, w, kp, ks);
      const int rbase = n_of(w) * N_PAIR;  // first replica of this pair tile
      const int m_blk = 2 * mp_of(w) + static_cast<int>(cr);
      k.inv = __frcp_rn(static_cast<float>(args.M - (args.t_begin + static_cast<uint64_t>(s))));
      const int buf = lt % NACC;
      // DIRECT: this tile's x, y, p rows (replica r, spins i0 .. i0+127: lane = spin) straight
      // from global memory, chunk c + 1 in flight while chunk c updates. The tile's dependency
      // (step s - 1 of its replica block complete, met before its MMAs could start) is acquired
      // here by every thread, so the loads are ordered after the writes they depend on.
      float dx[2][CWQ], dy[2][CWQ], dp[2][CWQ];
      const size_t dbase = static_cast<size_t>(rbase + h * CWQ) * args.npad + m_blk * Cfg::BM + srow;
      auto d_ld = [&](int c, int bb) {
#pragma unroll
        for (int j = 0; j < CWQ; ++j) {
          const size_t o = dbase + static_cast<size_t>(c * CW + j) * args.npad;
          dx[bb][j] = __ldcs(args.sx + o);
          dy[bb][j] = __ldcs(args.sy + o);
          dp[bb][j] = __ldcs(args.sp + o);
        }
      };
      if constexpr (Cfg::DIRECT) {
        if ((kp == ks - 1) && s > 0) dep::wait_block(args.done, n_of(w), args.done_base, s * args.num_m_total);
        if (kp == ks - 1) d_ld(0, 0);
      }
      if (SBG_DBG(args) < 2) ptx::mbar_wait(tfull_bar(buf), (lt / NACC) & 1);
      __syncwarp();
      ptx::tc_fence_after();
      const bool utr = SBG_HOOK_PTR(args.utrace) && lt < 64 && threadIdx.x == 4 * 32;
      auto ust = [&](int k) {
        if (utr) SBG_HOOK_PTR(args.utrace)[(static_cast<size_t>(blockIdx.x) * 64 + lt) * 8 + k] = gtimer_pair();
      };
      ust(2);
      if (utr) SBG_HOOK_PTR(args.utrace)[(static_cast<size_t>(blockIdx.x) * 64 + lt) * 8 + 6] = (uint64_t(s) << 40) | (uint64_t(w) << 8) | (uint64_t(kp) << 4) | uint64_t(ks);
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + buf * Cfg::ACC_COLS;
      // K split: partial fields of parts 0..KS-2, replica-major so a warp's 32 rows are contiguous
      const size_t frow = static_cast<size_t>(m_blk) * Cfg::BM + srow;
      auto fpart_at = [&](int part, int col) {
        return args.fpart + (static_cast<size_t>(part) * args.rpad + rbase + col) * args.npad + frow;
      };
      // the field of chunk c (this thread's CWQ replicas) from the accumulator columns
      auto load_F = [&](int c, float* F) {
        const int col0 = c * CW + h * CWQ;
        if constexpr (NA > 1) {
          // fixed-point real J: F = fl32(sum_w fl64(acc_w * 2^(8w + fx_exp))), fixed order (as step_tma.cuh)
          double f[CWQ];
#pragma unroll
          for (int j = 0; j < CWQ; ++j) f[j] = 0.0;
#pragma unroll
          for (int w = Cfg::W0; w < Cfg::NW; ++w) {
            uint32_t v[CWQ];
            ptx::tmem_ld<CWQ>(t_row + (w - Cfg::W0) * N_PAIR + col0, v);
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
          for (int j = 0; j < CWQ; ++j)  // s32 (int8 MMA) or the same integer in f32 (e2m1 MMA; exact)
            F[j] = Cfg::Q4 ? __uint_as_float(v[j]) : static_cast<float>(static_cast<int32_t>(v[j]));
        } else {
          long long tot[CWQ];
#pragma unroll
          for (int j = 0; j < CWQ; ++j) tot[j] = 0;
#pragma unroll
          for (int pl = 0; pl < NPLANES; ++pl) {
            uint32_t v[CWQ];
            const int col = Cfg::MERGED ? (col0 / Cfg::B_HALF) * NPLANES * Cfg::B_HALF + pl * Cfg::B_HALF +
                                              col0 % Cfg::B_HALF
                                        : pl * N_PAIR + col0;
            ptx::tmem_ld<CWQ>(t_row + col, v);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CWQ; ++j) tot[j] += static_cast<long long>(static_cast<int32_t>(v[j])) << (8 * pl);
          }
#pragma unroll
          for (int j = 0; j < CWQ; ++j) F[j] = __fmul_rn(__ll2float_rn(tot[j]), 0x1p-30f);
        }
      };
      if (NPLANES == 1 && ks > 1 && kp != ks - 1) {
        // a leading K part: publish the partial field, free the accumulator, count the part
#pragma unroll
        for (int c = 0; c < CHUNKS; ++c) {
          float F[CWQ];
          load_F(c, F);
#pragma unroll
          for (int j = 0; j < CWQ; ++j) __stcg(fpart_at(kp, c * CW + h * CWQ + j), F[j]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(buf ? tempty_leader1 : tempty_leader0);
        ptx::named_bar_sync(1, Cfg::EPI_WARPS * 32);
        if (threadIdx.x == 4 * 32) {
          __threadfence();
          dep::release_add(args.kdone + static_cast<size_t>(n_of(w)) * args.num_m + m_blk, 1u);
        }
        ust(4);
        continue;
      }
      if (NPLANES == 1 && ks > 1) {  // the last K part: wait for the other parts of this tile
        if (threadIdx.x == 4 * 32) {
          const uint32_t need = static_cast<uint32_t>((KS - 1) * (s + 1));
          const uint32_t* kd = args.kdone + static_cast<size_t>(n_of(w)) * args.num_m + m_blk;
          while (dep::ld_acquire(kd) < need) __nanosleep(32);
          __threadfence();
        }
        ptx::named_bar_sync(1, Cfg::EPI_WARPS * 32);
        ust(3);
      }
      float Fall[Cfg::EARLY_DRAIN ? CHUNKS : 1][CWQ];
      if constexpr (Cfg::EARLY_DRAIN) {  // one accumulator buffer: drain, release, then update
#pragma unroll
        for (int c = 0; c < CHUNKS; ++c) load_F(c, Fall[c]);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader0);
      }
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c, ++ck) {
        const int b = ck % NBUF;
        const int col0 = c * CW + h * CWQ;
        float F[CWQ];
        if constexpr (Cfg::EARLY_DRAIN) {
#pragma unroll
          for (int j = 0; j < CWQ; ++j) F[j] = Fall[c][j];
        } else {
          load_F(c, F);
        }
        if (NPLANES == 1 && ks > 1) {
          // exact integers below 2^24 (|F| <= kpad): fp32 sums in any order are exact
          for (int part = 0; part < ks - 1; ++part)
#pragma unroll
            for (int j = 0; j < CWQ; ++j) F[j] += __ldcg(fpart_at(part, col0 + j));
        }
        if constexpr (Cfg::DIRECT) {
          if (c + 1 < CHUNKS) d_ld(c + 1, (c + 1) & 1);
        }
        ptx::mbar_wait(sfull_bar(b), (ck / NBUF) & 1);
        float* xs = reinterpret_cast<float*>(s_gen + b * Cfg::BUF_BYTES);
        float* ys = xs + CW * Cfg::BM;
        float* ps = ys + CW * Cfg::BM;
        uint8_t* gs = reinterpret_cast<uint8_t*>(ps + CW * Cfg::BM);
#pragma unroll
        for (int j = 0; j < CWQ; ++j) {
          const int idx = (h * CWQ + j) * Cfg::BM + srow;
          float xv, yv, pv;
          if constexpr (Cfg::DIRECT) {
            xv = dx[c & 1][j], yv = dy[c & 1][j], pv = dp[c & 1][j];
          } else {
            xv = xs[idx], yv = ys[idx], pv = ps[idx];
          }
          PhaseConsts kj = k;
          if (args.a_rep) kj.a = args.a_rep[min(rbase + col0 + j, args.R - 1)];
          gsb_phase(F[j], xv, yv, pv, kj);
          if constexpr (Cfg::DIRECT) {
            const size_t o = dbase + static_cast<size_t>(c * CW + j) * args.npad;
            __stcs(args.sx + o, xv);
            __stcs(args.sy + o, yv);
            __stcs(args.sp + o, pv);
          } else {
            xs[idx] = xv;
            ys[idx] = yv;
            ps[idx] = pv;
          }
          if constexpr (Cfg::Q4) {
            // e2m1 codes (+1 = 0x2, -1 = 0xA) two spins per byte: lanes 2i, 2i+1 hold spins
            // 2i, 2i+1 of column j; the even lane writes the byte (warp-uniform shuffle)
            const uint32_t code = xv >= 0.0f ? 0x2u : 0xAu;
            const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, code, 1);
            if (!(lane & 1)) gs[(h * CWQ + j) * (Cfg::BM / 2) + (srow >> 1)] = static_cast<uint8_t>(code | (other << 4));
          } else if (NPLANES == 1) {
            gs[idx] = static_cast<uint8_t>(sgn8(xv));
          } else {
            const uint32_t qv = qdigits(quant30(xv));
#pragma unroll
            for (int pl = 0; pl < NPLANES; ++pl) gs[pl * Cfg::ST_G + idx] = static_cast<uint8_t>(qv >> (8 * pl));
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(sdone_bar(b));
      }
      ust(4);
      if constexpr (!Cfg::EARLY_DRAIN) {
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(buf ? tempty_leader1 : tempty_leader0);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();  // no remote arrive may target a CTA that has exited
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
}

}  // namespace sbg
