// The resident sign-variant kernel with each 160-replica block split into PARTS
// independent column parts whose step chains interleave (e2m1 operands).
//
// One step of one part is a chain of latencies: its G_t arrives from L2 -> MMAs ->
// epilogue -> G_{t+1} stored and released -> every CTA pair of the block has released ->
// the next G load. The communication links (store, release, the peers' releases, the
// load) cost ~2.5 us per step whatever the part width, the MMAs and the epilogue shrink
// with it; with PARTS chains in flight the tensor pipe and the epilogue warps work on one
// part while the others communicate. Each part has its own accumulator columns, G tile,
// done counter (done[PARTS n + i]) and handshakes.
//
// Per CTA TMEM (lane = spin of this CTA): [0, 160) f32 accumulators (part i at OFF[i]),
// [160, 320) x, [320, 480) y, [496, 512) unit E8M0 scale factors. p lives in the epilogue
// threads' registers (40 per thread). JRES (npad <= 2048): this CTA's 128 rows of J stay
// in shared memory for the launch (8 tiles of 16 KB e2m1) and the ring carries only G;
// otherwise each ring stage holds a J tile and a G tile.
// Warps: 0 operand producer, 1 MMA issuer (leader CTA), 2 TMEM allocator, 3 G publishers
// (lane i: TMA store of part i's G tile, completion wait, release of its counter), 4..19
// epilogue: warp (q = lane quadrant, cg = column group) owns columns
// OFF[i] + cg * W[i] / 4 + [0, W[i] / 4) of every part i.
// Arithmetic is gsb_phase2 on exact integer fields: bitwise equal to step_resident.cuh.
#pragma once

#include <cstdint>
#include <type_traits>
#include <utility>
#include <cuda.h>

#include "gsb_phase.cuh"
#include "ptx.cuh"
#include "step_resident.cuh"
#include "step_tma.cuh"

namespace sbg {

// Part widths (UMMA N, multiples of 16 for M = 256) of a 160-replica block.
template <int PARTS>
struct PartTable;
template <>
struct PartTable<2> {
  static constexpr int W[2] = {80, 80};
};
template <>
struct PartTable<3> {
  static constexpr int W[3] = {64, 48, 48};
};
template <>
struct PartTable<4> {
  static constexpr int W[4] = {48, 48, 32, 32};
};
template <>
struct PartTable<5> {
  static constexpr int W[5] = {32, 32, 32, 32, 32};
};

// Tensor maps of the parts kernel: G boxes depend on the part width (two width classes:
// class 0 = W[0], class 1 = the narrower parts).
struct PartMaps {
  CUtensorMap J;           // e2m1 J [npad][npad / 2], box 128 x 128 B, 128B swizzle
  CUtensorMap Gin[2][2];   // [class][step parity]: B operand [rpad][npad / 2], box W / 2 rows x 128 B
  CUtensorMap Gout[2][2];  // [class][step parity]: next G, [R][ceil(n / 2)], box W rows x 64 B
  CUtensorMap Gin3[2][2];  // JRES: the same B operand viewed [K block][rpad][128 B], box {128 B, W / 2, KB}:
                           // a part-step's whole G operand in one load
};

template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

template <int STAGES_, bool JRES_, int PARTS_>
struct PartsCfg {
  static constexpr int PARTS = PARTS_;
  static constexpr bool JRES = JRES_;
  using T = PartTable<PARTS>;
  __host__ __device__ static constexpr int w(int i) { return T::W[i]; }
  __host__ __device__ static constexpr int off(int i) { return i == 0 ? 0 : off(i - 1) + w(i - 1); }
  __host__ __device__ static constexpr int cls(int i) { return w(i) == w(0) ? 0 : 1; }
  static constexpr int BM = 128;                  // spins per CTA
  static constexpr int BK = 128;                  // K bytes per stage (256 e2m1 elements)
  static constexpr int NR = 160;                  // replicas per pair block
  static constexpr int J_SLOTS = JRES ? 8 : 0;    // resident J tiles (K <= 2048)
  static constexpr int A_BYTES = BM * BK;         // 16 KB
  static constexpr int B_BYTES = (w(0) / 2) * BK; // G rows of the widest part per CTA
  // JRES: a ring of STAGES super-stages, each holding a part-step's whole G operand (KB <= 8 K
  // blocks of W / 2 rows, one 3D TMA load and one barrier); else STAGES stages of (J tile, G tile)
  static constexpr int STAGE_BYTES = JRES ? J_SLOTS * B_BYTES : A_BYTES + B_BYTES;
  static constexpr int STAGES = STAGES_;
  static constexpr int RND = 4;                   // K-stages per MMA issue round
  static constexpr int EPI_WARPS = 16;
  static constexpr int CH = 4;                    // columns per TMEM load chunk
  static constexpr int T_BYTES = NR * BM / 2;     // G tiles of all parts: [160][64] bytes
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int NUM_BARS = 2 * STAGES + 4 * PARTS + 1;
  static constexpr int SMEM_BYTES = J_SLOTS * A_BYTES + STAGES * STAGE_BYTES + T_BYTES + 1024 + 8 * NUM_BARS + 64;
  static constexpr uint32_t COL_X = NR, COL_Y = 2 * NR, COL_SF = 512 - 16;
  static_assert(off(PARTS - 1) + w(PARTS - 1) == NR, "parts cover the block");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "SW128 stage alignment");
};

template <int STAGES_, bool JRES_, int PARTS_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PartsCfg<STAGES_, JRES_, PARTS_>::THREADS, 1)
    gsb_resident_parts_kernel(const __grid_constant__ PartMaps maps, const ResidentArgs args) {
  using Cfg = PartsCfg<STAGES_, JRES_, PARTS_>;
  constexpr int CH = Cfg::CH;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int PARTS = Cfg::PARTS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_addr);
  // JRES: [J_SLOTS] resident J tiles, then the G stages; else [STAGES] J tiles, [STAGES] G tiles
  const uint32_t a_base = base;
  const uint32_t b_base = base + (Cfg::JRES ? Cfg::J_SLOTS : STAGES) * Cfg::A_BYTES;
  const uint32_t t_base = base + Cfg::J_SLOTS * Cfg::A_BYTES + STAGES * Cfg::STAGE_BYTES;  // G tiles
  uint8_t* g_tile = smem + (t_base - base);
  uint64_t* bars = reinterpret_cast<uint64_t*>(g_tile + Cfg::T_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);
  // groups whose state the epilogue has loaded (paces the G_0 helper, warp 2)
  volatile int32_t* started = reinterpret_cast<volatile int32_t*>(tmem_slot + 1);
  auto bar = [&](int i) { return ptx::smem_u32(bars + i); };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(STAGES + s); };
  auto tfull_bar = [&](int i) { return bar(2 * STAGES + i); };              // accumulator i ready (both CTAs)
  auto tempty_bar = [&](int i) { return bar(2 * STAGES + PARTS + i); };     // accumulator i drained (leader)
  auto gfull_bar = [&](int i) { return bar(2 * STAGES + 2 * PARTS + i); };  // G tile i written (local)
  auto gempty_bar = [&](int i) { return bar(2 * STAGES + 3 * PARTS + i); }; // G tile i stored (local)
  const uint32_t jfull_bar = bar(2 * STAGES + 4 * PARTS);                   // JRES: J resident (leader)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cr = ptx::cluster_ctarank();
  const bool leader = cr == 0;
  // dev trace (SBG_RES_TRACE): %globaltimer stamps of pair 0's leader CTA, group 0, parts 0 and 1:
  // [s][part][k], k = 0 G dependency met, 6 first MMA round's stages landed, 7 all stages landed,
  // 1 accumulator ready (epilogue), 2 epilogue done, 3 publisher has the tile, 4 store complete,
  // 5 released, 8 producer issued all G loads, 9 MMAs issued
  // dev group trace (SBG_RES_GTRACE): k 0 group top, 1 state loaded, 2 step 0 part 0 acc ready,
  // 3 step 1 part 0 acc ready, 4 last step done, 5 write-back done, 6 helper published G_0
  auto gstamp = [&](int g, int k) {
    if (SBG_HOOK_PTR(args.gtrace) && g - args.group0 < 64)
      SBG_HOOK_PTR(args.gtrace)[(static_cast<size_t>(blockIdx.x) * 64 + (g - args.group0)) * 8 + k] = gtimer();
  };
  auto stamp = [&](int g, int s, int i, int k) {
    if (SBG_HOOK_PTR(args.trace) && g == args.group0 && s >= 0 && i < 2 && cr == 0 && (blockIdx.x >> 1) == 0)
      SBG_HOOK_PTR(args.trace)[(s * 2 + i) * 16 + k] = gtimer();
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(full_bar(s), 2);
      ptx::mbar_init(empty_bar(s), 1);
    }
    for (int i = 0; i < PARTS; ++i) {
      ptx::mbar_init(tfull_bar(i), 1);
      ptx::mbar_init(tempty_bar(i), 2 * Cfg::EPI_WARPS);
      ptx::mbar_init(gfull_bar(i), Cfg::EPI_WARPS);
      ptx::mbar_init(gempty_bar(i), 1);
    }
    ptx::mbar_init(jfull_bar, 2);
    ptx::fence_mbar_init();
    *started = 0;
  }
  if (warp == 2) {
    ptx::tmem_alloc_pair(ptx::smem_u32(tmem_slot), 512);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp >= 4 && warp < 8) {  // unit E8M0 scale factors (127 = 2^0)
    uint32_t v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
    const uint32_t t = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) + Cfg::COL_SF;
    ptx::tmem_st8(t, v);
    ptx::tmem_st8(t + 8, v);
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();

  const int num_mp = args.num_m / 2;
  const int pair = blockIdx.x >> 1;
  const int mp = pair % num_mp, rbk = pair / num_mp;
  const int m_blk = 2 * mp + static_cast<int>(cr);
  const int i0 = m_blk * Cfg::BM;
  const int KB = args.npad / (2 * Cfg::BK);
  const int num_n = (args.rpad + Cfg::NR - 1) / Cfg::NR;

  if (warp == 0) {  // ------------------------------------------------ operand producer
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&maps.J);
      for (int c = 0; c < 2; ++c)
        for (int p = 0; p < 2; ++p) ptx::prefetch_tmap(&maps.Gin[c][p]);
    }
    int stage = 0;
    uint32_t ph = 0;
    const uint64_t keep = ptx::policy_evict_last();
    if constexpr (Cfg::JRES) {  // this CTA's 128 rows of J, once per launch
      if (ptx::elect_one()) {
        const uint32_t fb = ptx::mapa(jfull_bar, 0);
        ptx::mbar_arrive_expect_tx_cluster(fb, KB * Cfg::A_BYTES);
        for (int kb = 0; kb < KB; ++kb)
          ptx::tma_load_2d_pair_hint(a_base + kb * Cfg::A_BYTES, &maps.J, fb, kb * Cfg::BK, m_blk * Cfg::BM, keep);
      }
      __syncwarp();
    }
    for (int g = args.group0; g < args.group0 + args.groups; ++g) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      for (int s = 0; s < args.nsteps; ++s) {
        static_for<0, PARTS>([&](auto I) {
          constexpr int i = decltype(I)::value;
          constexpr uint32_t b_bytes = (Cfg::w(i) / 2) * Cfg::BK;
          const CUtensorMap* gin = &maps.Gin[Cfg::cls(i)][s & 1];
          const int b_row0 = n_blk * Cfg::NR + Cfg::off(i) + static_cast<int>(cr) * (Cfg::w(i) / 2);
          // J tiles do not depend on the step: requested before the dependency wait
          int st0 = stage;
          uint32_t ph0 = ph;
          for (int kb = 0; !Cfg::JRES && kb < STAGES && kb < KB; ++kb) {
            ptx::mbar_wait(empty_bar(st0), ph0 ^ 1u);
            if (ptx::elect_one()) {
              const uint32_t fb = ptx::mapa(full_bar(st0), 0);
              ptx::mbar_expect_tx_cluster(fb, Cfg::A_BYTES);
              ptx::tma_load_2d_pair_hint(a_base + st0 * Cfg::A_BYTES, &maps.J, fb, kb * Cfg::BK, m_blk * Cfg::BM,
                                         keep);
            }
            __syncwarp();
            if (++st0 == STAGES) {
              st0 = 0;
              ph0 ^= 1u;
            }
          }
          // G_t of part i of block n: released by all num_m CTAs (G_0 by the kernel at group start).
          // (Per-producer-pair flags with the stages issued as their pairs become ready measured
          // slower: 34.0 vs 31.4 us/step at C2.)
          dep::wait_block(args.done, PARTS * n_blk + i, 0u, static_cast<uint32_t>((s + 1) * args.num_m));
          if (lane == 0) stamp(g, s, i, 0);
          if constexpr (Cfg::JRES) {  // the part-step's KB G tiles in one 3D load
            ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
            if (ptx::elect_one()) {
              const uint32_t fb = ptx::mapa(full_bar(stage), 0);
              ptx::mbar_arrive_expect_tx_cluster(fb, KB * b_bytes);
              ptx::tma_load_3d_pair_hint(b_base + stage * Cfg::STAGE_BYTES, &maps.Gin3[Cfg::cls(i)][s & 1], fb, 0,
                                         b_row0, 0, keep);
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              ph ^= 1u;
            }
          }
          for (int kb = 0; !Cfg::JRES && kb < KB; ++kb) {
            const bool pre = kb < STAGES;
            if (!pre) ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
            if (ptx::elect_one()) {
              const uint32_t fb = ptx::mapa(full_bar(stage), 0);
              ptx::mbar_arrive_expect_tx_cluster(fb, pre ? b_bytes : Cfg::A_BYTES + b_bytes);
              if (!pre)
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
          if (lane == 0) stamp(g, s, i, 8);
        });
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA issuer (leader)
    if (leader) {
      const uint32_t sf = tmem_base + Cfg::COL_SF;
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      if constexpr (Cfg::JRES) ptx::mbar_wait(jfull_bar, 0);
      for (int g = args.group0; g < args.group0 + args.groups; ++g) {
        const int n_blk = g * args.rb_per_group + rbk;
        if (n_blk >= num_n) break;
        for (int s = 0; s < args.nsteps; ++s, ++lt) {
          static_for<0, PARTS>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr uint32_t idesc = ptx::idesc_mxf4(256, Cfg::w(i));
            ptx::mbar_wait(tempty_bar(i), (lt & 1) ^ 1u);
            ptx::tc_fence_after();
            const uint32_t d = tmem_base + Cfg::off(i);
            if constexpr (Cfg::JRES) {  // one super-stage: all KB K blocks of this part-step
              ptx::mbar_wait(full_bar(stage), ph);
              if (lane == 0) {
                stamp(g, s, i, 6);
                stamp(g, s, i, 7);
              }
              ptx::tc_fence_after();
              if (ptx::elect_one()) {
                const uint32_t bb = b_base + stage * Cfg::STAGE_BYTES;
                const int kb_end = SBG_DBG(args) == 3 ? 2 : KB;  // dev timing probe: MMA cost off the chain
                for (int kb = 0; kb < kb_end; ++kb) {
                  const uint64_t adesc = ptx::smem_desc_k_sw128(a_base + kb * Cfg::A_BYTES);
                  const uint64_t bdesc = ptx::smem_desc_k_sw128(bb + kb * (Cfg::w(i) / 2) * Cfg::BK);
#pragma unroll
                  for (int k = 0; k < Cfg::BK / 32; ++k)
                    ptx::mma_mxf4_pair(d, adesc + 2 * k, bdesc + 2 * k, idesc, sf, (kb | k) != 0);
                }
                ptx::mma_commit_pair_mc(empty_bar(stage), 0x3);
              }
              __syncwarp();
              if (++stage == STAGES) {
                stage = 0;
                ph ^= 1u;
              }
            }
            // RND K-stages per issue round: one handshake (wait, fence, elect) per round
            constexpr int RND = Cfg::RND;
            for (int kb = 0; !Cfg::JRES && kb < KB; kb += RND) {
              int sts[RND];
              const int cnt = KB - kb < RND ? KB - kb : RND;
#pragma unroll
              for (int u = 0; u < RND; ++u) {
                if (u < cnt) {
                  ptx::mbar_wait(full_bar(stage), ph);
                  sts[u] = stage;
                  if (++stage == STAGES) {
                    stage = 0;
                    ph ^= 1u;
                  }
                }
              }
              if (lane == 0 && kb == 0) stamp(g, s, i, 6);
              if (lane == 0 && kb + RND >= KB) stamp(g, s, i, 7);
              ptx::tc_fence_after();
              if (ptx::elect_one()) {
#pragma unroll
                for (int u = 0; u < RND; ++u) {
                  if (u < cnt) {
                    const uint64_t adesc = ptx::smem_desc_k_sw128(a_base + sts[u] * Cfg::A_BYTES);
                    const uint64_t bdesc = ptx::smem_desc_k_sw128(b_base + sts[u] * Cfg::B_BYTES);
#pragma unroll
                    for (int k = 0; k < Cfg::BK / 32; ++k)
                      ptx::mma_mxf4_pair(d, adesc + 2 * k, bdesc + 2 * k, idesc, sf, (kb | u | k) != 0);
                    ptx::mma_commit_pair_mc(empty_bar(sts[u]), 0x3);
                  }
                }
              }
              __syncwarp();
            }
            if (ptx::elect_one()) ptx::mma_commit_pair_mc(tfull_bar(i), 0x3);
            __syncwarp();
            if (lane == 0) stamp(g, s, i, 9);
          });
        }
      }
    }
  } else if (warp == 2) {  // ------------------------------------------ G_0 helper
    // Group transitions off the critical path: while group g - 1 steps, publish group g's
    // G_0 = sgn(x_0) straight from global x (so its first MMAs can run while the epilogue is
    // still writing back g - 1 and loading g) and prefetch g's x, y, p rows into L2 (so that
    // load hits L2). Same bytes as the epilogue's put_g2 + the publisher's TMA store: row r <
    // R of the G buffer step 0 reads, bytes [i0 / 2, i0 / 2 + 64) clipped at (n + 1) / 2, two
    // spins per byte (even spin in the low nibble), +1 = 0x2, -1 = 0xA (sgn(0) = +1).
    const int64_t gpitch = args.npad / 2;
    const int gvalid = (args.n + 1) / 2;
    const int q = lane & 3;       // 32-spin chunk of this CTA's 128 spins
    const int b0 = i0 / 2 + q * 16;  // its first G byte
    for (int g = args.group0 + 1; g < args.group0 + args.groups; ++g) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      while (*started < g - args.group0) __nanosleep(256);  // group g - 1 under way here
      if (args.ready)
        while (dep::ld_acquire_sys(args.ready + args.rb_per_group + g - 1) == 0) __nanosleep(256);
      static_for<0, PARTS>([&](auto I) {
        constexpr int i = decltype(I)::value;
        const int r0 = n_blk * Cfg::NR + Cfg::off(i);
#pragma unroll 2
        for (int rr = lane >> 2; rr < Cfg::w(i); rr += 8) {
          const int r = r0 + rr;
          if (r >= args.R) continue;
          const float4* src = reinterpret_cast<const float4*>(args.x + static_cast<size_t>(r) * args.npad + i0 + q * 32);
          float4 f[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) f[v] = src[v];
          uint32_t w4[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            auto c = [](float xv) { return xv >= 0.0f ? 0x2u : 0xAu; };
            const float4 a = f[2 * v], b = f[2 * v + 1];
            w4[v] = c(a.x) | (c(a.y) << 4) | (c(a.z) << 8) | (c(a.w) << 12) | (c(b.x) << 16) | (c(b.y) << 20) |
                    (c(b.z) << 24) | (c(b.w) << 28);
          }
          uint8_t* dst = args.gbuf[1] + static_cast<size_t>(r) * gpitch + b0;
          if (b0 + 16 <= gvalid) {
            asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(w4[0]), "r"(w4[1]), "r"(w4[2]),
                         "r"(w4[3])
                         : "memory");
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (b0 + j < gvalid) dst[j] = static_cast<uint8_t>(w4[j >> 2] >> (8 * (j & 3)));
          }
        }
        // the consumers read G with TMA (async proxy) after acquiring the counter
        dep::fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) dep::release_add(args.done + PARTS * n_blk + i, 1u);
      });
      if (lane == 0) gstamp(g, 6);
      // L2 prefetch of the block's state rows (x was just read) for the epilogue's load
      for (int rr = lane; rr < Cfg::NR; rr += 32) {
        const int r = n_blk * Cfg::NR + rr;
        if (r >= args.rpad) break;
        const size_t off = static_cast<size_t>(r) * args.npad + i0;
        ptx::prefetch_l2_bulk(args.y + off, Cfg::BM * 4);
        ptx::prefetch_l2_bulk(args.p + off, Cfg::BM * 4);
        ptx::prefetch_l2_bulk(args.x + off, Cfg::BM * 4);
      }
    }
  } else if (warp == 3) {  // ------------------------------------------ G publishers
    // lane i publishes part i (its own bulk-async group, completion wait and release), so
    // the parts' store -> completion -> release latencies overlap instead of queueing
    if (lane < PARTS) {
      int offi = 0, clsi = 0;
      static_for<0, PARTS>([&](auto I) {
        constexpr int k = decltype(I)::value;
        if (lane == k) {
          offi = Cfg::off(k);
          clsi = Cfg::cls(k);
        }
      });
      if (lane == 0)
        for (int c = 0; c < 2; ++c)
          for (int p = 0; p < 2; ++p) ptx::prefetch_tmap(&maps.Gout[c][p]);
      int pc = 0;  // publishes so far
      for (int g = args.group0; g < args.group0 + args.groups; ++g) {
        const int n_blk = g * args.rb_per_group + rbk;
        if (n_blk >= num_n) break;
        // G_0 of the launch's first group (written by the state load into the buffer Gout[.][1]
        // writes; later groups' G_0 comes from the helper, warp 2), then G_{s+1}
        for (int s = g == args.group0 ? -1 : 0; s < args.nsteps; ++s, ++pc) {
          const int par = s < 0 ? 1 : (s & 1);
          ptx::mbar_wait(gfull_bar(lane), pc & 1);
          stamp(g, s, lane, 3);
          ptx::tma_store_2d(&maps.Gout[clsi][par], t_base + offi * (Cfg::BM / 2), i0 / 2, n_blk * Cfg::NR + offi);
          ptx::bulk_commit();
          ptx::bulk_wait_read0();
          ptx::mbar_arrive(gempty_bar(lane));  // tile reusable
          ptx::bulk_wait0();
          stamp(g, s, lane, 4);
          dep::fence_proxy_async_global();
          // red.release orders the completed (proxy-fenced) tile writes before the count
          dep::release_add(args.done + PARTS * n_blk + lane, 1u);
          stamp(g, s, lane, 5);
        }
      }
    }
  } else if (warp >= 4) {  // ----------------------------------------- epilogue
    const int q = warp & 3;
    const int cg = (warp - 4) >> 2;
    const int spin = i0 + q * 32 + lane;
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t g_sel = (lane & 1) ? 0x15u : 0x40u;
    float preg[Cfg::NR / 4];  // p of this thread's 40 columns: part i at off(i) / 4
    // e2m1 G codes of tile rows (row, row + 1), row even: lanes 2i, 2i+1 swap codes, the even
    // lane writes row's byte, the odd lane row + 1's (warp-uniform)
    auto put_g2 = [&](int row, float xa, float xb) {
      const uint32_t mine = (xa >= 0.0f ? 0x2u : 0xAu) | ((xb >= 0.0f ? 0x2u : 0xAu) << 8);
      const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, mine, 1);
      const uint32_t t = __byte_perm(mine, other, g_sel);
      g_tile[(row + (lane & 1)) * (Cfg::BM / 2) + ((spin - i0) >> 1)] = static_cast<uint8_t>(t | (t >> 4));
    };
    auto tile_written = [&](int i) {
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(gfull_bar(i));
    };
    int lt = 0, pc = 0;
    for (int g = args.group0; g < args.group0 + args.groups; ++g) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      if (args.ready)
        while (dep::ld_acquire_sys(args.ready + (g == 0 ? rbk : args.rb_per_group + g - 1)) == 0)
          __nanosleep(256);
      // load the block's state (x, y to TMEM, p to registers); for the launch's first group also
      // write G_0 = sgn(x_0) (later groups: published ahead by the helper, warp 2)
      const bool first = g == args.group0;
      const bool gt = warp == 4 && lane == 0;
      if (gt) gstamp(g, 0);
      // x, y to TMEM, p to registers, one 4-column chunk at a time
      static_for<0, PARTS>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int CHUNKS = Cfg::w(i) / 16;
        if (first) ptx::mbar_wait(gempty_bar(i), (pc & 1) ^ 1u);
        static_for<0, CHUNKS>([&](auto C) {
          constexpr int c = decltype(C)::value;
          const int col = Cfg::off(i) + cg * (Cfg::w(i) / 4) + c * CH;
          uint32_t vx[4], vy[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = n_blk * Cfg::NR + col + j;
            const size_t off = static_cast<size_t>(r) * args.npad + spin;
            const bool in = r < args.rpad;
            vx[j] = in ? __float_as_uint(args.x[off]) : 0u;
            vy[j] = in ? __float_as_uint(args.y[off]) : 0u;
            preg[Cfg::off(i) / 4 + c * CH + j] = in ? args.p[off] : 0.0f;
          }
          ptx::tmem_st<4>(t_lane + Cfg::COL_X + col, vx);
          ptx::tmem_st<4>(t_lane + Cfg::COL_Y + col, vy);
          if (first) {
            put_g2(col, __uint_as_float(vx[0]), __uint_as_float(vx[1]));
            put_g2(col + 2, __uint_as_float(vx[2]), __uint_as_float(vx[3]));
          }
        });
      });
      ptx::tmem_st_wait();
      if (first) {
        static_for<0, PARTS>([&](auto I) { tile_written(decltype(I)::value); });
        ++pc;
      }
      if (gt) {
        *started = g - args.group0 + 1;
        gstamp(g, 1);
      }
      for (int s = 0; s < args.nsteps; ++s, ++lt, ++pc) {
        PhaseConsts k = args.k;
        k.inv = __frcp_rn(static_cast<float>(args.M - (args.t_begin + static_cast<uint64_t>(s))));
        const PhaseConsts2 k2(k, args.ident);
        const float* arep = args.a_rep;
        // the previous step's x, y stores must land before this step re-reads those columns;
        // within a step every column is loaded once, so one wait per step covers all parts
        ptx::tmem_st_wait();
        static_for<0, PARTS>([&](auto I) {
          constexpr int i = decltype(I)::value;
          constexpr int CHUNKS = Cfg::w(i) / 16;
          const int c0 = Cfg::off(i) + cg * (Cfg::w(i) / 4);  // this warp's first column of part i
          uint32_t bf[2][CH], bx[2][CH], by[2][CH];
          auto ld_chunk = [&](int c, int b) {
            const uint32_t col = c0 + c * CH;
            ptx::tmem_ld<CH>(t_lane + col, bf[b]);
            ptx::tmem_ld<CH>(t_lane + Cfg::COL_X + col, bx[b]);
            ptx::tmem_ld<CH>(t_lane + Cfg::COL_Y + col, by[b]);
          };
          auto wait_chunk = [&](int b) {
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CH; ++j) asm volatile("" : "+r"(bf[b][j]), "+r"(bx[b][j]), "+r"(by[b][j]));
          };
          // x, y of the first chunk do not depend on the MMA: requested before its completion
          ptx::tmem_ld<CH>(t_lane + Cfg::COL_X + c0, bx[0]);
          ptx::tmem_ld<CH>(t_lane + Cfg::COL_Y + c0, by[0]);
          ptx::mbar_wait(tfull_bar(i), lt & 1);
          __syncwarp();
          ptx::tc_fence_after();
          const bool tr = warp == 4 && lane == 0;
          if (tr) stamp(g, s, i, 1);
          if (tr && i == 0 && s < 2) gstamp(g, 2 + s);
          ptx::mbar_wait(gempty_bar(i), (pc & 1) ^ 1u);  // this part's G tile stored
          if (tr) stamp(g, s, i, 10);
          ptx::tmem_ld<CH>(t_lane + c0, bf[0]);
          wait_chunk(0);
          if (tr) stamp(g, s, i, 11);
          auto chunks = [&](auto has_arep) {
            static_for<0, CHUNKS>([&](auto C) {
              constexpr int c = decltype(C)::value;
              constexpr int b = c & 1;
              if constexpr (c + 1 < CHUNKS) ld_chunk(c + 1, b ^ 1);
              const int col = c0 + c * CH;
#pragma unroll
              for (int j = 0; j < CH; j += 2) {
                float x0 = __uint_as_float(bx[b][j]), x1 = __uint_as_float(bx[b][j + 1]);
                float y0 = __uint_as_float(by[b][j]), y1 = __uint_as_float(by[b][j + 1]);
                float& p0 = preg[Cfg::off(i) / 4 + c * CH + j];
                float& p1 = preg[Cfg::off(i) / 4 + c * CH + j + 1];
                uint64_t a2 = k2.a;
                if constexpr (decltype(has_arep)::value) {
                  const int r = n_blk * Cfg::NR + col + j;
                  a2 = f2::pk(arep[min(r, args.R - 1)], arep[min(r + 1, args.R - 1)]);
                }
                // the field: the exact integer in f32 (e2m1 MMA)
                gsb_phase2(__uint_as_float(bf[b][j]), __uint_as_float(bf[b][j + 1]), x0, x1, y0, y1, p0, p1, k2, a2);
                bx[b][j] = __float_as_uint(x0);
                bx[b][j + 1] = __float_as_uint(x1);
                by[b][j] = __float_as_uint(y0);
                by[b][j + 1] = __float_as_uint(y1);
                put_g2(col + j, x0, x1);
              }
              ptx::tmem_st<CH>(t_lane + Cfg::COL_X + col, bx[b]);
              ptx::tmem_st<CH>(t_lane + Cfg::COL_Y + col, by[b]);
              if constexpr (c + 1 < CHUNKS) wait_chunk(b ^ 1);
            });
          };
          if (arep)
            chunks(std::true_type{});
          else
            chunks(std::false_type{});
          if (tr) stamp(g, s, i, 12);
          tile_written(i);  // first: the publisher stores G_{t+1} of part i and releases its counter
          // accumulator i consumed (all F loads waited): the leader may issue this part's next MMAs
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(tempty_bar(i), 0));
          if (tr) stamp(g, s, i, 2);
        });
      }
      // write the block's state back (after the last step's TMEM stores)
      if (gt) gstamp(g, 4);
      ptx::tmem_st_wait();
      const uint64_t wb_policy = ptx::policy_evict_first();  // written once, read by a later launch
      static_for<0, PARTS>([&](auto I) {
        constexpr int i = decltype(I)::value;
        static_for<0, Cfg::w(i) / 16>([&](auto C) {
          constexpr int c = decltype(C)::value;
          const int col = Cfg::off(i) + cg * (Cfg::w(i) / 4) + c * CH;
          uint32_t vx[4], vy[4];
          ptx::tmem_ld<4>(t_lane + Cfg::COL_X + col, vx);
          ptx::tmem_ld<4>(t_lane + Cfg::COL_Y + col, vy);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int r = n_blk * Cfg::NR + col + j;
            if (r >= args.rpad) continue;
            const size_t off = static_cast<size_t>(r) * args.npad + spin;
            ptx::st_hint(args.x + off, vx[j], wb_policy);
            ptx::st_hint(args.y + off, vy[j], wb_policy);
            ptx::st_hint(args.p + off, __float_as_uint(preg[Cfg::off(i) / 4 + c * CH + j]), wb_policy);
          }
        });
      });
      if (gt) gstamp(g, 5);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, 512);
}

}  // namespace sbg
