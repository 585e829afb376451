// Resident-state kernel, ping-pong variant: each CTA pair keeps TWO 64-replica
// blocks (A, B) resident in TMEM and alternates them, so that while one block is
// in its epilogue / G_{t+1} exchange / dependency wait, the tensor cores run the
// other block's contraction.
//
// step_resident.cuh serialises, per step, MMA (~2.1 us) -> epilogue (~2.2 us) ->
// publish (~1.35 us) -> wait for the other CTAs of the replica block; with two
// independent blocks the MMA of one block hides most of the other's chain.
// Per CTA TMEM (512 columns x 128 lanes, lane = spin):
//   [0,64) F_A  [64,128) F_B  [128,320) x_A y_A p_A  [320,512) x_B y_B p_B
// The operand ring carries (J tile, G_t half tile of the block) stages in the
// issue order (s,A), (s,B), (s+1,A), ...; J does not depend on the step, so its
// tiles are requested before the dependency wait of each block-step. All 16
// epilogue warps process one block at a time (16 replica columns per thread);
// warp 3 publishes each block's G_{t+1} tile (TMA store, then release done[n])
// while the epilogue warps move on to the other block.
// Arithmetic: gsb_phase2 (bitwise gsb_phase), as step_resident.cuh.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda.h>

#include "step_resident.cuh"

namespace sbg {

template <int STAGES_>
struct Res2Cfg {
  static constexpr int BM = 128;
  static constexpr int BK = 128;
  static constexpr int NR = 64;                  // replicas per block (UMMA N)
  static constexpr int NB = 2;                   // blocks per pair
  static constexpr int B_HALF = NR / 2;          // B rows staged per CTA
  static constexpr int A_BYTES = BM * BK;        // 16 KB
  static constexpr int B_BYTES = B_HALF * BK;    // 4 KB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = STAGES_;
  static constexpr int G_BYTES = NR * BM;        // one block's G_{t+1} tile [64 replicas][128 spins]
  static constexpr int EPI_WARPS = 16;
  static constexpr int COLS = NR / (EPI_WARPS / 4);  // 16 replica columns per epilogue thread
  static constexpr int CH = 4;
  static constexpr int CHUNKS = COLS / CH;
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int NUM_BARS = 2 * STAGES + 4;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + NB * G_BYTES + 1024 + 8 * NUM_BARS + 64;
  __host__ __device__ static constexpr uint32_t acc(int b) { return uint32_t(b * NR); }
  __host__ __device__ static constexpr uint32_t col_x(int b) { return uint32_t(2 * NR + b * 3 * NR); }
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

template <int STAGES_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Res2Cfg<STAGES_>::THREADS, 1)
    gsb_resident_pp_kernel(const __grid_constant__ TmaMaps maps, const ResidentArgs args) {
  using Cfg = Res2Cfg<STAGES_>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int NR = Cfg::NR;
  constexpr int CH = Cfg::CH;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_addr);
  const uint32_t a_base = base;
  const uint32_t b_base = base + STAGES * Cfg::A_BYTES;
  const uint32_t g_base = base + STAGES * Cfg::STAGE_BYTES;
  uint8_t* g_tile = smem + STAGES * Cfg::STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(g_tile + Cfg::NB * Cfg::G_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);
  auto bar = [&](int i) { return ptx::smem_u32(bars + i); };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(STAGES + s); };
  auto tfull = [&](int b) { return bar(2 * STAGES + b); };
  auto tempty = [&](int b) { return bar(2 * STAGES + 2 + b); };

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
      ptx::mbar_init(tfull(b), 1);
      ptx::mbar_init(tempty(b), 2 * Cfg::EPI_WARPS);
    }
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

  const int num_mp = args.num_m / 2;
  const int pair = blockIdx.x >> 1;
  const int mp = pair % num_mp, rbk = pair / num_mp;
  const int m_blk = 2 * mp + static_cast<int>(cr);
  const int i0 = m_blk * Cfg::BM;
  const int KB = args.npad / Cfg::BK;
  const int num_n = args.rpad / NR;  // 64-replica blocks
  // block X of pair-block bb of group g: replica block n = 2 * (g * rb_per_group + rbk) + X
  auto blk = [&](int g, int X) { return 2 * (g * args.rb_per_group + rbk) + X; };

  if (warp == 0) {  // ------------------------------------------------ operand producer
    if (ptx::elect_one()) {
      ptx::prefetch_tmap(&maps.J);
      ptx::prefetch_tmap(&maps.Gin[0]);
      ptx::prefetch_tmap(&maps.Gin[1]);
    }
    int stage = 0;
    uint32_t ph = 0;
    const uint64_t keep = ptx::policy_evict_last();
    constexpr int PRE = STAGES < 16 ? STAGES : 16;
    for (int g = 0; g < args.groups; ++g) {
      if (blk(g, 0) >= num_n) break;
      for (int s = 0; s < args.nsteps; ++s) {
        for (int X = 0; X < 2; ++X) {
          const int n_blk = blk(g, X);
          int st0 = stage;
          uint32_t ph0 = ph;
          const bool noload = args.dbg == 3 && (s > 0 || g > 0);
          for (int kb = 0; kb < PRE && kb < KB; ++kb) {
            ptx::mbar_wait(empty_bar(st0), ph0 ^ 1u);
            if (ptx::elect_one() && !noload) {
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
          if (n_blk < num_n && args.dbg < 2)
            dep::wait_block(args.done, n_blk, 0u, static_cast<uint32_t>(s * args.num_m));
          if (args.trace && pair == 0 && cr == 0 && g == 0 && lane == 0) args.trace[(s * 2 + X) * 8 + 0] = gtimer();
          const CUtensorMap* gin = &maps.Gin[s & 1];
          for (int kb = 0; kb < KB; ++kb) {
            const bool pre = kb < PRE;
            if (!pre) ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
            if (ptx::elect_one()) {
              const uint32_t fb = ptx::mapa(full_bar(stage), 0);
              ptx::mbar_arrive_expect_tx_cluster(fb, noload ? 0 : (pre ? Cfg::B_BYTES : Cfg::STAGE_BYTES));
              if (!pre && !noload)
                ptx::tma_load_2d_pair_hint(a_base + stage * Cfg::A_BYTES, &maps.J, fb, kb * Cfg::BK, m_blk * Cfg::BM,
                                           keep);
              if (!noload)
                ptx::tma_load_2d_pair_hint(b_base + stage * Cfg::B_BYTES, gin, fb, kb * Cfg::BK,
                                           n_blk * NR + static_cast<int>(cr) * Cfg::B_HALF, keep);
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              ph ^= 1u;
            }
          }
        }
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA issuer (leader)
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_i8(256, NR, true, true);
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int g = 0; g < args.groups; ++g) {
        if (blk(g, 0) >= num_n) break;
        for (int s = 0; s < args.nsteps; ++s, ++lt) {
          for (int X = 0; X < 2; ++X) {
            ptx::mbar_wait(tempty(X), (lt & 1) ^ 1u);
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
                  for (int k = 0; k < Cfg::BK / 32; ++k)
                    ptx::mma_i8_pair(tmem_base + Cfg::acc(X), adesc + 2 * k, bdesc + 2 * k, idesc, (kb | u | k) != 0);
                  ptx::mma_commit_pair_mc(empty_bar(st), 0x3);
                }
              }
              __syncwarp();
            }
            if (ptx::elect_one()) ptx::mma_commit_pair_mc(tfull(X), 0x3);
            __syncwarp();
          }
        }
      }
    }
  } else if (warp == 3) {  // ------------------------------------------ G publisher
    for (int g = 0; g < args.groups; ++g) {
      if (blk(g, 0) >= num_n) break;
      if (g > 0) ptx::named_bar_sync(6, 32 * (Cfg::EPI_WARPS + 1));  // previous group's tiles stored
      for (int s = 0; s < args.nsteps; ++s)
        for (int X = 0; X < 2; ++X) {
          ptx::named_bar_sync(2 + X, 32 * (Cfg::EPI_WARPS + 1));
          if (lane == 0) {
            const int n_blk = blk(g, X);
            ptx::tma_store_2d(&maps.Gout[s & 1], g_base + X * Cfg::G_BYTES, i0, n_blk * NR);
            ptx::bulk_commit();
            ptx::bulk_wait0();
            dep::fence_proxy_async_global();
            __threadfence();
            dep::release_add(args.done + n_blk, 1u);
            if (args.trace && pair == 0 && cr == 0 && g == 0) args.trace[(s * 2 + X) * 8 + 3] = gtimer();
          }
          __syncwarp();
        }
    }
  } else if (warp >= 4) {  // ----------------------------------------- epilogue (all blocks)
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;  // replica columns h*16 .. h*16+15 of the current block
    const int spin = i0 + q * 32 + lane;
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t tempty_leader[2] = {ptx::mapa(tempty(0), 0), ptx::mapa(tempty(1), 0)};
    int lt = 0;
    for (int g = 0; g < args.groups; ++g) {
      if (blk(g, 0) >= num_n) break;
      // g_tile may be rewritten only after the publisher's last stores of the previous group
      if (g > 0) ptx::named_bar_sync(6, 32 * (Cfg::EPI_WARPS + 1));
      // load both blocks' state into TMEM (a warp reads 32 consecutive spins per replica)
      for (int X = 0; X < 2; ++X) {
        const int r0 = blk(g, X) * NR + h * Cfg::COLS;
        uint32_t vx[16], vy[16], vp[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const size_t off = static_cast<size_t>(r0 + j) * args.npad + spin;
          vx[j] = __float_as_uint(args.x[off]);
          vy[j] = __float_as_uint(args.y[off]);
          vp[j] = __float_as_uint(args.p[off]);
        }
        const uint32_t col = Cfg::col_x(X) + h * Cfg::COLS;
        ptx::tmem_st16(t_lane + col, vx);
        ptx::tmem_st16(t_lane + col + NR, vy);
        ptx::tmem_st16(t_lane + col + 2 * NR, vp);
      }
      ptx::tmem_st_wait();
      for (int s = 0; s < args.nsteps; ++s, ++lt) {
        PhaseConsts k = args.k;
        k.inv = __frcp_rn(static_cast<float>(args.M - (args.t_begin + static_cast<uint64_t>(s))));
        const PhaseConsts2 k2(k, args.ident);
        const float* arep = args.a_rep;
        for (int X = 0; X < 2; ++X) {
          const int r0 = blk(g, X) * NR + h * Cfg::COLS;
          ptx::mbar_wait(tfull(X), lt & 1);
          __syncwarp();
          ptx::tc_fence_after();
          const bool tr = args.trace && pair == 0 && cr == 0 && g == 0 && threadIdx.x == 128;
          if (tr) args.trace[(s * 2 + X) * 8 + 1] = gtimer();
          uint8_t* gt = g_tile + X * Cfg::G_BYTES;
          uint32_t bf[2][CH], bx[2][CH], by[2][CH], bp[2][CH];
          const uint32_t ca = Cfg::acc(X) + h * Cfg::COLS, cx = Cfg::col_x(X) + h * Cfg::COLS;
          auto ld_chunk = [&](int c, int b) {
            ptx::tmem_ld<CH>(t_lane + ca + c * CH, bf[b]);
            ptx::tmem_ld<CH>(t_lane + cx + c * CH, bx[b]);
            ptx::tmem_ld<CH>(t_lane + cx + NR + c * CH, by[b]);
            ptx::tmem_ld<CH>(t_lane + cx + 2 * NR + c * CH, bp[b]);
          };
          auto wait_chunk = [&](int b) {
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < CH; ++j)
              asm volatile("" : "+r"(bf[b][j]), "+r"(bx[b][j]), "+r"(by[b][j]), "+r"(bp[b][j]));
          };
          ld_chunk(0, 0);
          wait_chunk(0);
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
                gsb_phase2(static_cast<float>(static_cast<int32_t>(bf[b][j])),
                           static_cast<float>(static_cast<int32_t>(bf[b][j + 1])), x0, x1, y0, y1, p0, p1, k2, a2);
                bx[b][j] = __float_as_uint(x0);
                bx[b][j + 1] = __float_as_uint(x1);
                by[b][j] = __float_as_uint(y0);
                by[b][j + 1] = __float_as_uint(y1);
                bp[b][j] = __float_as_uint(p0);
                bp[b][j + 1] = __float_as_uint(p1);
                uint8_t* gp = gt + (h * Cfg::COLS + c * CH + j) * Cfg::BM + q * 32 + lane;
                gp[0] = static_cast<uint8_t>(sgn8(x0));
                gp[Cfg::BM] = static_cast<uint8_t>(sgn8(x1));
              }
              ptx::tmem_st<CH>(t_lane + cx + c * CH, bx[b]);
              ptx::tmem_st<CH>(t_lane + cx + NR + c * CH, by[b]);
              ptx::tmem_st<CH>(t_lane + cx + 2 * NR + c * CH, bp[b]);
              if (c + 1 < Cfg::CHUNKS) wait_chunk(b ^ 1);
            }
          };
          if (arep)
            chunks(std::true_type{});
          else
            chunks(std::false_type{});
          ptx::tmem_st_wait();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader[X]);
          if (tr) args.trace[(s * 2 + X) * 8 + 2] = gtimer();
          ptx::fence_proxy_async_smem();
          asm volatile("bar.arrive %0, %1;" ::"r"(2 + X), "r"(32 * (Cfg::EPI_WARPS + 1)) : "memory");
        }
      }
      // write both blocks' state back
      for (int X = 0; X < 2; ++X) {
        const int r0 = blk(g, X) * NR + h * Cfg::COLS;
        const uint32_t col = Cfg::col_x(X) + h * Cfg::COLS;
        uint32_t vx[16], vy[16], vp[16];
        ptx::tmem_ld<16>(t_lane + col, vx);
        ptx::tmem_ld<16>(t_lane + col + NR, vy);
        ptx::tmem_ld<16>(t_lane + col + 2 * NR, vp);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const size_t off = static_cast<size_t>(r0 + j) * args.npad + spin;
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
