// The hot path with the replica state RESIDENT in tensor memory (sign variants).
//
// The streaming kernels (step_tma.cuh, step_pair.cuh) move x, y, p through HBM
// every step: 24 B per spin-update, which bounds C2 at ~60 us/step. Here each
// CTA pair owns a fixed (256-spin pair-block, 128-replica block) for a whole
// group of replicas and keeps that block's x, y, p in TMEM next to its
// accumulator, so the only per-step traffic is the operands from L2 (J rows and
// the G_t tile) and the 16 KB G_{t+1} chunk it publishes. HBM sees the state
// once per launch per group (load at group start, store at group end).
//
// Per CTA TMEM (512 columns x 128 lanes; lane = spin of this CTA):
//   [0, 128)    s32 accumulator F = J G_t for the 128 replicas of the block
//   [128, 256)  x     [256, 384) y     [384, 512) p      (fp32)
// Work decomposition: pairs are arranged num_mp (spin pair-blocks) x RB
// (replica blocks per group); replica block of group g is n = g*RB + rbk.
// Groups run one after another inside the launch; every pair of a group runs
// all nsteps steps of its block. Step t+1 of block n needs G_{t+1}[n] from all
// num_m CTAs of the block: the done[n] counters of step_tma.cuh (released after
// each CTA's G chunk store completes, acquired by the operand producers).
// Warps: 0 operand producer (both CTAs), 1 MMA issuer (leader), 2 TMEM
// allocator, 3 idle, 4..19 epilogue (4 per TMEM lane quadrant, 32 replica
// columns each): tcgen05.ld F and state, gsb_phase, tcgen05.st state, sign
// bytes into a 16 KB smem tile, one TMA store of the tile, release done[n].
// Arithmetic is the streaming kernels' gsb_phase, so results are bitwise equal.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda.h>

#include "gsb_phase.cuh"
#include "ptx.cuh"
#include "step_tma.cuh"

namespace sbg {

namespace ptx {
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&v)[N]);
template <>
__device__ __forceinline__ void tmem_st<4>(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
template <>
__device__ __forceinline__ void tmem_st<8>(uint32_t taddr, const uint32_t (&v)[8]) {
  tmem_st8(taddr, v);
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
}  // namespace ptx

// NR_ = replicas per pair block (UMMA N). 128: F, x, y, p all in TMEM (4 x 128 columns);
// 160: F, x, y in TMEM (480 columns) and p in shared memory ([160][128] fp32, 80 KB),
// which takes 25% more replicas per group (fewer sequential groups per step).
// Q4_: operands as packed e2m1 (two K elements per byte, even element in the low nibble):
// J entries in {0, +-1, +-2, +-3, +-4, +-6} and G = +-1 are exact in e2m1, so
// tcgen05.mma.kind::mxf4.block_scale with unit (E8M0 = 127) scales accumulates the
// same integer field in fp32 (exact: |F| < 2^24), at twice the int8 MMA rate and half
// the operand bytes (tools/dev/mxf4_probe.cu). The unit scales take SF_COLS TMEM columns.
template <int STAGES_, int EPI_WARPS_ = 16, int CH_ = 4, int NR_ = 128, bool GD_ = false, bool Q4_ = false>
struct ResCfg {
  static constexpr bool Q4 = Q4_;
  static constexpr int BM = 128;                 // spins per CTA
  static constexpr int BK = 128;                 // K bytes per stage (128 int8 / 256 e2m1 elements)
  static constexpr int KPB = Q4 ? 2 : 1;         // K elements per byte
  static constexpr int NR = NR_;                 // replicas per pair block (UMMA N)
  static constexpr int SF_COLS = Q4 ? 16 : 0;    // unit scale factors (last TMEM columns)
  static constexpr uint32_t COL_SF = 512 - SF_COLS;
  static constexpr bool P_SMEM = 4 * NR + SF_COLS > 512;  // part of p leaves TMEM
  static constexpr int P_T = P_SMEM ? 512 - SF_COLS - 3 * NR : NR;  // p columns kept in TMEM (the rest in smem)
  static constexpr int B_HALF = NR / 2;          // B rows staged per CTA
  static constexpr int A_BYTES = BM * BK;        // 16 KB
  static constexpr int B_BYTES = B_HALF * BK;    // 8 KB (NR 128)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = STAGES_;
  // G_{t+1} staging tile [NR][128] for one TMA store; G_DIRECT: the epilogue stores the sign
  // bytes straight to global memory instead (frees the tile's shared memory for a ring stage)
  static constexpr bool G_DIRECT = GD_;
  static constexpr int G_BYTES = G_DIRECT ? 0 : NR * BM / KPB;
  static constexpr int P_BYTES = (NR - P_T) * BM * 4;
  static constexpr int EPI_WARPS = EPI_WARPS_;           // 4 per TMEM lane quadrant x column groups
  static constexpr int COLS_PER_WARP = NR / (EPI_WARPS / 4);
  static constexpr int CH = CH_;                           // replica columns per TMEM load chunk
  static constexpr int CHUNKS = COLS_PER_WARP / CH;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int NUM_BARS = 2 * STAGES + 2;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + G_BYTES + P_BYTES + 1024 + 8 * NUM_BARS + 64;
  static constexpr uint32_t COL_X = NR, COL_Y = 2 * NR, COL_P = 3 * NR;  // p: [COL_P, COL_P + P_T)
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(NR % 16 == 0 && NR <= 256 && COLS_PER_WARP % 8 == 0, "UMMA N / epilogue chunking");
  static_assert(3 * NR + P_T + SF_COLS <= 512 && P_T % 4 == 0, "TMEM columns");
  // p of a warp's column block: its first PT_W columns in TMEM, the rest in shared memory
  // (balanced over the column groups so no epilogue warp does more TMEM traffic)
  static constexpr int PT_W = P_T / (EPI_WARPS / 4);
  static_assert((PT_W % 4 == 0 && CH_ % 4 == 0) || !P_SMEM, "p split granularity");
  static_assert(!(Q4 && G_DIRECT), "e2m1 G is published through the smem tile");
};

struct ResidentArgs {
  int32_t n, npad, R, rpad;
  int32_t num_m;     // 128-spin blocks (CTAs per replica block)
  int32_t rb_per_group;
  int32_t group0;    // first replica group of this launch
  int32_t groups;    // groups in this launch
  PhaseConsts k;
  uint64_t M, t_begin;
  int32_t nsteps;
  uint32_t* done;    // [rpad / 128], zero at launch
  float *x, *y, *p;  // replica-major [rpad][npad]
  const float* a_rep;
  PhaseIdent ident;           // -0, 1, -1 (runtime identity operands of gsb_phase2)
  uint8_t* gbuf[2];           // G_DIRECT: output G buffer of step parity 0/1 ([rpad][npad] bytes)
  const uint32_t* ready;      // optional: nonzero once the x, y rows have landed (sbg_run overlaps the
                              // host->device copies with the steps): [0, rb_per_group) the blocks of
                              // group 0, then one flag per later group (rb_per_group + g - 1)
  int32_t dbg;                // dev only: 1 = skip J loads after the first step, 2 = no G dependency wait
  unsigned long long* trace;  // dev only: per-step %globaltimer stamps of pair 0 (null = off)
  unsigned long long* gtrace; // dev only: per-(CTA, group) stamps of the parts kernel [cta][64][8]
  const uint8_t* j4;          // TS kernel: packed e2m1 J [npad][npad / 2] (rows loaded into TMEM)
  int64_t j4_pitch;           // its row pitch in bytes
  int32_t trace_group;        // dev only: the launch-relative group SBG_RES_TRACE stamps (SBG_RES_TRACE - 1)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int STAGES_, int EPI_WARPS_, int CH_, int NR_, bool Q4_ = false>
__global__ void __cluster_dims__(2, 1, 1)
    __launch_bounds__(ResCfg<STAGES_, EPI_WARPS_, CH_, NR_, false, Q4_>::THREADS, 1)
        gsb_resident_pair_kernel(const __grid_constant__ TmaMaps maps, const ResidentArgs args) {
  using Cfg = ResCfg<STAGES_, EPI_WARPS_, CH_, NR_, false, Q4_>;
  constexpr int CH = Cfg::CH;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_addr);
  const uint32_t a_base = base;
  const uint32_t b_base = base + STAGES * Cfg::A_BYTES;
  const uint32_t g_base = base + STAGES * Cfg::STAGE_BYTES;
  uint8_t* g_tile = smem + STAGES * Cfg::STAGE_BYTES;
  float* p_smem = reinterpret_cast<float*>(g_tile + Cfg::G_BYTES);  // p columns >= P_T: [NR - P_T][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(g_tile + Cfg::G_BYTES + Cfg::P_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);
  auto bar = [&](int i) { return ptx::smem_u32(bars + i); };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(STAGES + s); };
  const uint32_t tfull = bar(2 * STAGES), tempty = bar(2 * STAGES + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cr = ptx::cluster_ctarank();
  const bool leader = cr == 0;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), 2);
      ptx::mbar_init(empty_bar(s), 1);
    }
    ptx::mbar_init(tfull, 1);
    ptx::mbar_init(tempty, 2 * Cfg::EPI_WARPS);
    ptx::fence_mbar_init();
  }
  if (warp == 2) {
    ptx::tmem_alloc_pair(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if constexpr (Cfg::Q4) {  // unit E8M0 scale factors (127 = 2^0) in the last SF_COLS columns
    if (warp >= 4 && warp < 8) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
      const uint32_t t = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + Cfg::COL_SF;
#pragma unroll
      for (int c = 0; c < Cfg::SF_COLS; c += 8) ptx::tmem_st8(t + c, v);
      ptx::tmem_st_wait();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    ptx::tc_fence_after();
  }

  const int num_mp = args.num_m / 2;
  const int pair = blockIdx.x >> 1;
  const int mp = pair % num_mp, rbk = pair / num_mp;
  const int m_blk = 2 * mp + static_cast<int>(cr);
  const int i0 = m_blk * Cfg::BM;
  const int KB = args.npad / (Cfg::BK * Cfg::KPB);
  const int num_n = (args.rpad + Cfg::NR - 1) / Cfg::NR;  // the last block may pass rpad (NR 160)

  if (warp == 0) {  // ------------------------------------------------ operand producer
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&maps.J);
      ptx::prefetch_tmap(&maps.Gin[0]);
      ptx::prefetch_tmap(&maps.Gin[1]);
    }
    int stage = 0;
    uint32_t ph = 0;
    const uint64_t keep = ptx::policy_evict_last();
    for (int g = args.group0; g < args.group0 + args.groups; ++g) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      const int b_row0 = n_blk * Cfg::NR + static_cast<int>(cr) * Cfg::B_HALF;  // this CTA's B rows
      for (int s = 0; s < args.nsteps; ++s) {
        // J does not depend on the step: the first PRE stages' J tiles are requested
        // before waiting for G_t (expect_tx without arrive), the G halves after.
        constexpr int PRE = STAGES < 16 ? STAGES : 16;
        int st0 = stage;
        uint32_t ph0 = ph;
        const bool skipJ = SBG_DBG(args) == 1 && (s > 0 || g > 0);
        for (int kb = 0; kb < PRE && kb < KB; ++kb) {
          ptx::mbar_wait(empty_bar(st0), ph0 ^ 1u);
          if (ptx::elect_one() && !skipJ) {
            const uint32_t fb = ptx::mapa(full_bar(st0), 0);
            ptx::mbar_expect_tx_cluster(fb, Cfg::A_BYTES);
            ptx::tma_load_2d_pair_hint(a_base + st0 * Cfg::A_BYTES, &maps.J, fb, kb * Cfg::BK, m_blk * Cfg::BM, keep);
          }
          __syncwarp();
          if (++st0 == STAGES) {
            st0 = 0;
            ph0 ^= 1u;
          }
        }
        // G_t of block n is complete when all num_m CTAs released it (the launch's
        // initial G_0 is published by the kernel itself at group start: one release each)
        if (SBG_DBG(args) != 2) dep::wait_block(args.done, n_blk, 0u, static_cast<uint32_t>((s + 1) * args.num_m));
        if (SBG_HOOK_PTR(args.trace) && pair == 0 && g == 0 && lane == 0) SBG_HOOK_PTR(args.trace)[(s * 2 + cr) * 16 + 0] = gtimer();
        const CUtensorMap* gin = &maps.Gin[s & 1];
        for (int kb = 0; kb < KB; ++kb) {
          const bool pre = kb < PRE;
          if (!pre) ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
          if (ptx::elect_one()) {
            const uint32_t fb = ptx::mapa(full_bar(stage), 0);
            ptx::mbar_arrive_expect_tx_cluster(fb, (pre || skipJ) ? Cfg::B_BYTES : Cfg::STAGE_BYTES);
            if (!pre && !skipJ)
              ptx::tma_load_2d_pair_hint(a_base + stage * Cfg::A_BYTES, &maps.J, fb, kb * Cfg::BK, m_blk * Cfg::BM,
                                         keep);
            ptx::tma_load_2d_pair_hint(b_base + stage * Cfg::B_BYTES, gin, fb, kb * Cfg::BK, b_row0, keep);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA issuer (leader)
    if (leader) {
      constexpr uint32_t idesc = Cfg::Q4 ? ptx::idesc_mxf4(256, Cfg::NR) : ptx::idesc_i8(256, Cfg::NR, true, true);
      const uint32_t sf = tmem_base + Cfg::COL_SF;
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int g = args.group0; g < args.group0 + args.groups; ++g) {
        const int n_blk = g * args.rb_per_group + rbk;
        if (n_blk >= num_n) break;
        for (int s = 0; s < args.nsteps; ++s, ++lt) {
          ptx::mbar_wait(tempty, (lt & 1) ^ 1u);
          ptx::tc_fence_after();
          // two K-stages per issue round: the per-round handshake (wait, fence, elect,
          // commit) costs ~260 cycles, more than 4 MMAs of N <= 128 (tools/dev/pipe_probe.cu)
          for (int kb = 0; kb < KB; kb += 2) {
            const int st0 = stage;
            ptx::mbar_wait(full_bar(stage), ph);
            if (++stage == STAGES) {
              stage = 0;
              ph ^= 1u;
            }
            const int st1 = stage;
            const bool two = kb + 1 < KB;
            if (two) {
              ptx::mbar_wait(full_bar(stage), ph);
              if (++stage == STAGES) {
                stage = 0;
                ph ^= 1u;
              }
            }
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                if (u == 1 && !two) break;
                const int st = u ? st1 : st0;
                const uint64_t adesc = ptx::smem_desc_k_sw128(a_base + st * Cfg::A_BYTES);
                const uint64_t bdesc = ptx::smem_desc_k_sw128(b_base + st * Cfg::B_BYTES);
#pragma unroll
                for (int k = 0; k < Cfg::BK / 32; ++k) {  // 32 bytes per MMA (K = 32 int8 / 64 e2m1)
                  if constexpr (Cfg::Q4)
                    ptx::mma_mxf4_pair(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, sf, (kb | u | k) != 0);
                  else
                    ptx::mma_i8_pair(tmem_base, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | u | k) != 0);
                }
                ptx::mma_commit_pair_mc(empty_bar(st), 0x3);
              }
            }
            __syncwarp();
          }
          if (ptx::elect_one()) ptx::mma_commit_pair_mc(tfull, 0x3);
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {  // ----------------------------------------- epilogue
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const int spin = i0 + q * 32 + lane;
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t tempty_leader = ptx::mapa(tempty, 0);
    const int epi_tid = threadIdx.x - 128;
    // G_{t+1} byte of (replica column col of the block, this thread's spin): smem tile, or
    // straight to the global buffer of step parity par (bounded like the TMA store: R x n)
    auto put_g = [&](int n_blk, int col, int par, float xv) {
      if constexpr (Cfg::G_DIRECT) {
        const int r = n_blk * Cfg::NR + col;
        if (r < args.R && spin < args.n)
          args.gbuf[par][static_cast<size_t>(r) * args.npad + spin] = static_cast<uint8_t>(sgn8(xv));
      } else {
        g_tile[col * Cfg::BM + (spin - i0)] = static_cast<uint8_t>(sgn8(xv));
      }
    };
    // G_{t+1} of columns (col, col + 1), col even: int8 bytes, or for Q4 e2m1 codes (+1 = 0x2,
    // -1 = 0xA) packed two spins per byte; lanes 2i, 2i+1 (spins 2i, 2i+1) swap codes so the
    // even lane writes column col's byte and the odd lane column col + 1's. Warp-uniform.
    const uint32_t g_sel = (lane & 1) ? 0x15u : 0x40u;
    auto put_g2 = [&](int n_blk, int col, int par, float xa, float xb) {
      if constexpr (Cfg::Q4) {
        const uint32_t mine = (xa >= 0.0f ? 0x2u : 0xAu) | ((xb >= 0.0f ? 0x2u : 0xAu) << 8);
        const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, mine, 1);
        // even lane: (its code, partner's code) of column col; odd: (partner's, its) of col + 1
        const uint32_t t = __byte_perm(mine, other, g_sel);
        g_tile[(col + (lane & 1)) * (Cfg::BM / 2) + ((spin - i0) >> 1)] = static_cast<uint8_t>(t | (t >> 4));
      } else {
        put_g(n_blk, col, par, xa);
        put_g(n_blk, col + 1, par, xb);
      }
    };
    // publish this CTA's G chunk of block n_blk for the consumers of step parity par
    auto publish = [&](int n_blk, int par) {
      if constexpr (Cfg::G_DIRECT) {
        __threadfence();
        ptx::named_bar_sync(1, 32 * Cfg::EPI_WARPS);
        if (epi_tid == 0) {
          dep::fence_proxy_async_global();
          dep::release_add(args.done + n_blk, 1u);
        }
      } else {
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, 32 * Cfg::EPI_WARPS);
        if (epi_tid == 0) {
          ptx::tma_store_2d(&maps.Gout[par], g_base, i0 / Cfg::KPB, n_blk * Cfg::NR);
          ptx::bulk_commit();
          ptx::bulk_wait0();
          dep::fence_proxy_async_global();
          __threadfence();
          dep::release_add(args.done + n_blk, 1u);
        }
        ptx::named_bar_sync(1, 32 * Cfg::EPI_WARPS);  // g_tile reusable
      }
    };
    int lt = 0;
    for (int g = args.group0; g < args.group0 + args.groups; ++g) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      const int r0 = n_blk * Cfg::NR + h * Cfg::COLS_PER_WARP;  // this thread's first replica
      if (args.ready)
        while (dep::ld_acquire_sys(args.ready + (g == 0 ? rbk : args.rb_per_group + g - 1)) == 0)
          __nanosleep(256);
      // load the block's state into TMEM (coalesced: a warp reads 32 consecutive spins)
#pragma unroll 1
      for (int c8 = 0; c8 < Cfg::COLS_PER_WARP / 8; ++c8) {
        uint32_t vx[8], vy[8], vp[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = r0 + c8 * 8 + j;
          const size_t off = static_cast<size_t>(r) * args.npad + spin;
          const bool in = r < args.rpad;  // the last block of a non-dividing NR may pass rpad
          vx[j] = in ? __float_as_uint(args.x[off]) : 0u;
          vy[j] = in ? __float_as_uint(args.y[off]) : 0u;
          vp[j] = in ? __float_as_uint(args.p[off]) : 0u;
        }
        const uint32_t col = h * Cfg::COLS_PER_WARP + c8 * 8;
        ptx::tmem_st<8>(t_lane + Cfg::COL_X + col, vx);
        ptx::tmem_st<8>(t_lane + Cfg::COL_Y + col, vy);
#pragma unroll
        for (int u = 0; u < 8; u += 4) {  // p in units of 4 columns: TMEM below PT_W, else smem
          const int c4 = c8 * 8 + u;
          if (c4 < Cfg::PT_W) {
            const uint32_t v4[4] = {vp[u], vp[u + 1], vp[u + 2], vp[u + 3]};
            ptx::tmem_st<4>(t_lane + Cfg::COL_P + h * Cfg::PT_W + c4, v4);
          } else {
            const int ps = h * (Cfg::COLS_PER_WARP - Cfg::PT_W) + c4 - Cfg::PT_W;
#pragma unroll
            for (int j = 0; j < 4; ++j) p_smem[(ps + j) * Cfg::BM + q * 32 + lane] = __uint_as_float(vp[u + j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; j += 2) put_g2(n_blk, col + j, 1, __uint_as_float(vx[j]), __uint_as_float(vx[j + 1]));
      }
      ptx::tmem_st_wait();
      // publish G_0 = sgn(x) of this block (the B operand of the launch's first step:
      // the buffer Gout[1] writes), so a launch needs no host-side preparation
      publish(n_blk, 1);
      for (int s = 0; s < args.nsteps; ++s, ++lt) {
        PhaseConsts k = args.k;
        k.inv = __frcp_rn(static_cast<float>(args.M - (args.t_begin + static_cast<uint64_t>(s))));
        const PhaseConsts2 k2(k, args.ident);
        const float* arep = args.a_rep;
        ptx::mbar_wait(tfull, lt & 1);
        __syncwarp();
        ptx::tc_fence_after();
        if (SBG_HOOK_PTR(args.trace) && pair == 0 && g == 0 && epi_tid == 0) SBG_HOOK_PTR(args.trace)[(s * 2 + cr) * 16 + 1] = gtimer();
        // chunks of CH replica columns; TMEM loads of chunk c+1 overlap the math of chunk c
        uint32_t bf[2][CH], bx[2][CH], by[2][CH], bp[2][CH];
        auto ld_chunk = [&](int c, int b) {
          const uint32_t col = h * Cfg::COLS_PER_WARP + c * CH;
          ptx::tmem_ld<CH>(t_lane + col, bf[b]);
          ptx::tmem_ld<CH>(t_lane + Cfg::COL_X + col, bx[b]);
          ptx::tmem_ld<CH>(t_lane + Cfg::COL_Y + col, by[b]);
          if (c * CH < Cfg::PT_W) {
            ptx::tmem_ld<CH>(t_lane + Cfg::COL_P + h * Cfg::PT_W + c * CH, bp[b]);
          } else {
            const int ps = h * (Cfg::COLS_PER_WARP - Cfg::PT_W) + c * CH - Cfg::PT_W;
#pragma unroll
            for (int j = 0; j < CH; ++j) bp[b][j] = __float_as_uint(p_smem[(ps + j) * Cfg::BM + q * 32 + lane]);
          }
        };
        auto wait_chunk = [&](int b) {
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < CH; ++j) asm volatile("" : "+r"(bf[b][j]), "+r"(bx[b][j]), "+r"(by[b][j]), "+r"(bp[b][j]));
        };
        ld_chunk(0, 0);
        wait_chunk(0);
        const bool tr = SBG_HOOK_PTR(args.trace) && pair == 0 && g == 0 && epi_tid == 0;
        if (tr) SBG_HOOK_PTR(args.trace)[(s * 2 + cr) * 16 + 4] = gtimer();
        auto chunks = [&](auto has_arep) {
#pragma unroll
          for (int c = 0; c < Cfg::CHUNKS; ++c) {
            const int b = c & 1;
            if (c + 1 < Cfg::CHUNKS) ld_chunk(c + 1, b ^ 1);
#pragma unroll
            for (int j = 0; j < CH; j += 2) {
              float x0 = __uint_as_float(bx[b][j]), x1 = __uint_as_float(bx[b][j + 1]);
              float y0 = __uint_as_float(by[b][j]), y1 = __uint_as_float(by[b][j + 1]);
              float p0 = __uint_as_float(bp[b][j]), p1 = __uint_as_float(bp[b][j + 1]);
              uint64_t a2 = k2.a;
              if constexpr (decltype(has_arep)::value)
                a2 = f2::pk(arep[min(r0 + c * CH + j, args.R - 1)], arep[min(r0 + c * CH + j + 1, args.R - 1)]);
              // the field: s32 (int8 MMA) or the same integer in f32 (e2m1 MMA; exact)
              const float f0 = Cfg::Q4 ? __uint_as_float(bf[b][j]) : static_cast<float>(static_cast<int32_t>(bf[b][j]));
              const float f1 =
                  Cfg::Q4 ? __uint_as_float(bf[b][j + 1]) : static_cast<float>(static_cast<int32_t>(bf[b][j + 1]));
              gsb_phase2(f0, f1, x0, x1, y0, y1, p0, p1, k2, a2);
              bx[b][j] = __float_as_uint(x0);
              bx[b][j + 1] = __float_as_uint(x1);
              by[b][j] = __float_as_uint(y0);
              by[b][j + 1] = __float_as_uint(y1);
              bp[b][j] = __float_as_uint(p0);
              bp[b][j + 1] = __float_as_uint(p1);
              put_g2(n_blk, h * Cfg::COLS_PER_WARP + c * CH + j, s & 1, x0, x1);
            }
            const uint32_t col = h * Cfg::COLS_PER_WARP + c * CH;
            ptx::tmem_st<CH>(t_lane + Cfg::COL_X + col, bx[b]);
            ptx::tmem_st<CH>(t_lane + Cfg::COL_Y + col, by[b]);
            if (c * CH < Cfg::PT_W) {
              ptx::tmem_st<CH>(t_lane + Cfg::COL_P + h * Cfg::PT_W + c * CH, bp[b]);
            } else {
              const int ps = h * (Cfg::COLS_PER_WARP - Cfg::PT_W) + c * CH - Cfg::PT_W;
#pragma unroll
              for (int j = 0; j < CH; ++j) p_smem[(ps + j) * Cfg::BM + q * 32 + lane] = __uint_as_float(bp[b][j]);
            }
            if (c + 1 < Cfg::CHUNKS) wait_chunk(b ^ 1);
          }
        };
        if (arep)
          chunks(std::true_type{});
        else
          chunks(std::false_type{});
        if (tr) SBG_HOOK_PTR(args.trace)[(s * 2 + cr) * 16 + 5] = gtimer();
        ptx::tmem_st_wait();
        if (tr) SBG_HOOK_PTR(args.trace)[(s * 2 + cr) * 16 + 6] = gtimer();
        // F consumed: the leader may overwrite the accumulator
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader);
        // publish G_{t+1} for this CTA's 128 spins x NR replicas
        if (tr) SBG_HOOK_PTR(args.trace)[(s * 2 + cr) * 16 + 2] = gtimer();
        publish(n_blk, s & 1);
        if (tr) SBG_HOOK_PTR(args.trace)[(s * 2 + cr) * 16 + 3] = gtimer();
      }
      // write the block's state back
#pragma unroll 1
      for (int c8 = 0; c8 < Cfg::COLS_PER_WARP / 8; ++c8) {
        const uint32_t col = h * Cfg::COLS_PER_WARP + c8 * 8;
        uint32_t vx[8], vy[8], vp[8], vp4[2][4];
        ptx::tmem_ld<8>(t_lane + Cfg::COL_X + col, vx);
        ptx::tmem_ld<8>(t_lane + Cfg::COL_Y + col, vy);
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (c8 * 8 + 4 * u < Cfg::PT_W) ptx::tmem_ld<4>(t_lane + Cfg::COL_P + h * Cfg::PT_W + c8 * 8 + 4 * u, vp4[u]);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c4 = c8 * 8 + 4 * u;
          const int ps = h * (Cfg::COLS_PER_WARP - Cfg::PT_W) + c4 - Cfg::PT_W;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            vp[4 * u + j] = c4 < Cfg::PT_W ? vp4[u][j] : __float_as_uint(p_smem[(ps + j) * Cfg::BM + q * 32 + lane]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int r = r0 + c8 * 8 + j;
          if (r >= args.rpad) continue;
          const size_t off = static_cast<size_t>(r) * args.npad + spin;
          args.x[off] = __uint_as_float(vx[j]);
          args.y[off] = __uint_as_float(vy[j]);
          args.p[off] = __uint_as_float(vp[j]);
        }
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, 512);
}

}  // namespace sbg
