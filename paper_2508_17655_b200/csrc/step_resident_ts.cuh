// The resident sign-variant kernel with J in TENSOR MEMORY (A operand of a "TS" MMA) and the
// replica state x, y in shared memory (e2m1 operands, npad <= 2048).
//
// Why: in the parts kernel (step_resident_parts.cuh) every part-step's MMAs re-read this
// CTA's 128 rows of J (16 KB per K block) from shared memory as the A operand. For the
// narrow parts that interleave the step chains (N = 48 / 32) that read, not the math, paces
// the tensor pipe: 41 / 39 cycles per M=256, K=64 kind::mxf4 instruction against the N/2 =
// 24 / 16 cycle floor (tools/dev/mxf4_ts_probe.cu, measured on the B200). With A in TMEM
// (tcgen05.mma ... [d], [a_tmem], b_desc: UTCOMMA tmem[..], gdesc[..]) the same
// instructions run at the floor, so each part's MMAs finish in half the time and the step
// chain shortens by that much. J takes 256 TMEM columns (K = 2048 e2m1, 8 per 32-bit
// column; lane = row), so x and y move to shared memory ([160 replicas][128 spins] fp32
// each, the layout a 2D TMA box of the replica-major state lands in): group transitions
// become two TMA loads / two TMA stores per CTA instead of per-thread loads and stores.
//
// Per CTA TMEM: [0, 160) f32 accumulators (part i at OFF[i]), [160, 416) J (e2m1, K block
// kb at columns 160 + 32 kb), [496, 512) unit E8M0 scale factors. Shared memory: x, y
// (80 KB each), STAGES G super-stages, the parts' G tiles. p stays in the epilogue threads'
// registers. Warps and the step protocol are those of the parts kernel: 0 G producer,
// 1 MMA issuer (leader CTA), 2 TMEM allocator then G_0 helper for later groups, 3 G
// publishers, 4..19 epilogue. Arithmetic is gsb_phase2 on exact integer fields: results
// are bitwise those of the parts kernel (tests/test_gpu_parity.py).
#pragma once

#include <cstdint>
#include <cuda.h>

#include "gsb_phase.cuh"
#include "ptx.cuh"
#include "step_resident.cuh"
#include "step_resident_parts.cuh"
#include "step_tma.cuh"

#ifndef SBG_TS_PPART
#define SBG_TS_PPART 0  // 1: p written back / loaded part by part in a group's last step
#endif
#ifndef SBG_TS_REGS
#define SBG_TS_REGS 0  // dev: 1 = setmaxnreg moves registers from warps 0..3 (48) to the epilogue warps (104)
#endif
#ifndef SBG_TS_TRACE4
#define SBG_TS_TRACE4 0  // 1: SBG_RES_TRACE stamps all four parts (tools/dev/trace_parts4.py), dev builds only
#endif
#ifndef SBG_TS_LD1
#define SBG_TS_LD1 0  // 1: one TMEM load + wait per part-step (measured the same, 26.6 us; spills 36 B)
#endif

namespace sbg {

namespace ptx {
__device__ __forceinline__ void mma_mxf4_pair_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t sf_tmem, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sf_tmem)
      : "memory");
}
__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
}  // namespace ptx

// Tensor maps of the TS kernel: the parts kernel's G maps plus the state boxes.
struct TsMaps {
  PartMaps g;
  CUtensorMap Gin3h[2][2];  // KH2: the 3D G view with box depth KB / 2 (a part-step's G in two halves)
  CUtensorMap X[2], Y[2];  // f32 [rpad][npad], box {128 spins, part width} per width class
};

// PKB_: per-K-block dependencies. Each K block of a part's G operand (256 spins = one CTA
// pair's slab) has its own done counter, TMA load and mbarrier, and the MMA warp issues the
// K blocks' MMAs in the order they land (exact integer sums: any order gives the same field),
// so a part's MMAs overlap the wait for the slowest of the 16 producer CTAs instead of
// starting after it.
// KH2_: a part-step's G operand in two 3D loads (K blocks [0, KB/2) and [KB/2, KB)) on two
// barriers, so the first half's MMAs run while the second half is in flight.
template <int STAGES_, int PARTS_, bool PKB_ = false, bool KH2_ = false>
struct TsCfg {
  static constexpr bool PKB = PKB_;
  static constexpr bool KH2 = KH2_;
  static constexpr int PARTS = PARTS_;
  using T = PartTable<PARTS>;
  __host__ __device__ static constexpr int w(int i) { return T::W[i]; }
  __host__ __device__ static constexpr int off(int i) { return i == 0 ? 0 : off(i - 1) + w(i - 1); }
  __host__ __device__ static constexpr int cls(int i) { return w(i) == w(0) ? 0 : 1; }
  static constexpr int BM = 128;                   // spins per CTA
  static constexpr int BK = 128;                   // K bytes per K block (256 e2m1 elements)
  static constexpr int NR = 160;                   // replicas per pair block
  static constexpr int KB_MAX = 8;                 // K blocks (npad <= 2048)
  static constexpr int B_BYTES = (w(0) / 2) * BK;  // G rows of the widest part per CTA, one K block
  static constexpr int STAGE_BYTES = KB_MAX * B_BYTES;  // a part-step's whole G operand (one 3D load)
  static constexpr int STAGES = STAGES_;
  static constexpr int EPI_WARPS = 16;
  static constexpr int CH = 4;                     // columns per chunk
  static constexpr int XY_BYTES = NR * BM * 4;     // 80 KB each
  static constexpr int T_BYTES = NR * BM / 2;      // G tiles of all parts: [160][64] bytes
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int NUM_BARS = 2 * STAGES + 5 * PARTS + (PKB ? STAGES * KB_MAX : 0) + (KH2 ? STAGES : 0);
  static constexpr int SMEM_BYTES = 2 * XY_BYTES + STAGES * STAGE_BYTES + T_BYTES + 1024 + 8 * NUM_BARS + 64;
  static constexpr uint32_t COL_J = NR, COL_SF = 512 - 16;
  static_assert(off(PARTS - 1) + w(PARTS - 1) == NR, "parts cover the block");
  static_assert(COL_J + 32 * KB_MAX <= COL_SF, "TMEM columns");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(STAGE_BYTES % 1024 == 0 && XY_BYTES % 1024 == 0, "alignment");
  static_assert(!(PKB && KH2), "one G load scheme");
};

template <int STAGES_, int PARTS_, bool PKB_, bool KH2_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TsCfg<STAGES_, PARTS_, PKB_, KH2_>::THREADS, 1)
    gsb_resident_ts_kernel(const __grid_constant__ TsMaps maps, const ResidentArgs args) {
  using Cfg = TsCfg<STAGES_, PARTS_, PKB_, KH2_>;
  constexpr int CH = Cfg::CH;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int PARTS = Cfg::PARTS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = ptx::smem_u32(smem_raw);
  const uint32_t base = (raw_addr + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_addr);
  const uint32_t x_base = base;                          // x [NR][BM] f32
  const uint32_t y_base = base + Cfg::XY_BYTES;          // y [NR][BM] f32
  const uint32_t b_base = base + 2 * Cfg::XY_BYTES;      // G super-stages
  const uint32_t t_base = b_base + STAGES * Cfg::STAGE_BYTES;  // G tiles
  uint8_t* g_tile = smem + (t_base - base);
  uint64_t* bars = reinterpret_cast<uint64_t*>(g_tile + Cfg::T_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + Cfg::NUM_BARS);
  volatile int32_t* started = reinterpret_cast<volatile int32_t*>(tmem_slot + 1);
  auto bar = [&](int i) { return ptx::smem_u32(bars + i); };
  auto full_bar = [&](int s) { return bar(s); };
  auto empty_bar = [&](int s) { return bar(STAGES + s); };
  auto tfull_bar = [&](int i) { return bar(2 * STAGES + i); };
  auto tempty_bar = [&](int i) { return bar(2 * STAGES + PARTS + i); };
  auto gfull_bar = [&](int i) { return bar(2 * STAGES + 2 * PARTS + i); };
  auto gempty_bar = [&](int i) { return bar(2 * STAGES + 3 * PARTS + i); };
  auto sfull_bar = [&](int i) { return bar(2 * STAGES + 4 * PARTS + i); };  // part i's x, y landed (TMA)
  auto fullk_bar = [&](int st, int kb) { return bar(2 * STAGES + 5 * PARTS + st * Cfg::KB_MAX + kb); };  // PKB
  auto full2_bar = [&](int st) { return bar(2 * STAGES + 5 * PARTS + st); };  // KH2: second half (first: full_bar)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cr = ptx::cluster_ctarank();
  const bool leader = cr == 0;
  // dev trace (SBG_RES_TRACE): the parts kernel's per-step stamps (pair 0 leader, group 0, parts 0, 1)
  auto stamp = [&](int g, int s, int i, int k) {
    if constexpr (!SBG_DEVHOOKS) return;
    // parts 0, 1 in the parts kernel's layout; SBG_TS_TRACE4 builds also stamp parts 2, 3 into a
    // second region of the same shape (compile-time: stamps in all four parts' loops change the
    // register allocation of this kernel and cost 4 % even with the trace off)
    if (SBG_HOOK_PTR(args.trace) && g == args.group0 + args.trace_group && s >= 0 && i < (SBG_TS_TRACE4 ? 4 : 2) && cr == 0 &&
        (blockIdx.x >> 1) == 0)
      SBG_HOOK_PTR(args.trace)[((i >> 1) * 2 * 4096 + s * 2 + (i & 1)) * 16 + k] = gtimer();
  };
  auto gstamp = [&](int g, int k) {
    if constexpr (!SBG_DEVHOOKS) return;
    if (SBG_HOOK_PTR(args.gtrace) && g - args.group0 < 64)
      SBG_HOOK_PTR(args.gtrace)[(static_cast<size_t>(blockIdx.x) * 64 + (g - args.group0)) * 8 + k] = gtimer();
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
    for (int i = 0; i < PARTS; ++i) ptx::mbar_init(sfull_bar(i), 1);
    if constexpr (Cfg::PKB)
      for (int st = 0; st < STAGES; ++st)
        for (int kb = 0; kb < Cfg::KB_MAX; ++kb) ptx::mbar_init(fullk_bar(st, kb), 2);
    if constexpr (Cfg::KH2)
      for (int st = 0; st < STAGES; ++st) ptx::mbar_init(full2_bar(st), 2);
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

  const int num_mp = args.num_m / 2;
  const int pair = blockIdx.x >> 1;
  const int mp = pair % num_mp, rbk = pair / num_mp;
  const int m_blk = 2 * mp + static_cast<int>(cr);
  const int i0 = m_blk * Cfg::BM;
  const int KB = args.npad / (2 * Cfg::BK);
  const int num_n = (args.rpad + Cfg::NR - 1) / Cfg::NR;
  // done counter a CTA releases for (block, part): per (block, part) counting all num_m CTAs,
  // or with PKB per (block, part, CTA pair) counting the pair's 2 CTAs
  auto done_idx = [&](int n_blk, int i) { return Cfg::PKB ? (n_blk * PARTS + i) * num_mp + mp : PARTS * n_blk + i; };

  if (warp >= 4) {
    // unit E8M0 scale factors, and this CTA's 128 rows of J into TMEM: lane = row, K block kb at
    // columns COL_J + 32 kb, the packed row's bytes as little-endian 32-bit words (8 e2m1 each,
    // even element in the low nibble: the layout the TS MMA reads, mxf4_ts_probe.cu)
    const int q = warp & 3, cg = (warp - 4) >> 2;
    const uint32_t tl = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    if (cg == 0) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
      ptx::tmem_st8(tl + Cfg::COL_SF, v);
      ptx::tmem_st8(tl + Cfg::COL_SF + 8, v);
    }
    const uint4* row = reinterpret_cast<const uint4*>(args.j4 + static_cast<size_t>(i0 + q * 32 + lane) * args.j4_pitch);
    for (int c = cg * 16; c < KB * 32; c += 64) {  // 16 columns (64 B) per store, column group cg
      uint32_t v[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint4 w4 = row[c / 4 + u];
        v[4 * u] = w4.x;
        v[4 * u + 1] = w4.y;
        v[4 * u + 2] = w4.z;
        v[4 * u + 3] = w4.w;
      }
      ptx::tmem_st16(tl + Cfg::COL_J + c, v);
    }
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();

#if SBG_TS_REGS
  if (warp < 4) {
    ptx::setmaxnreg_dec<48>();
#endif
  if (warp == 0) {  // ------------------------------------------------ G producer
    if (ptx::elect_one())
      for (int c = 0; c < 2; ++c)
        for (int p = 0; p < 2; ++p) {
          ptx::prefetch_tmap(&maps.g.Gin3[c][p]);
          ptx::prefetch_tmap(&maps.g.Gin[c][p]);
        }
    int stage = 0;
    uint32_t ph = 0;
    const uint64_t keep = ptx::policy_evict_last();
    for (int g = args.group0; g < args.group0 + args.groups; ++g) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      for (int s = 0; s < args.nsteps; ++s) {
        static_for<0, PARTS>([&](auto I) {
          constexpr int i = decltype(I)::value;
          constexpr uint32_t b_bytes = (Cfg::w(i) / 2) * Cfg::BK;
          const int b_row0 = n_blk * Cfg::NR + Cfg::off(i) + static_cast<int>(cr) * (Cfg::w(i) / 2);
          if constexpr (Cfg::PKB) {
            // lane kb: wait for producer pair kb's slab of G_s, then load it (its own barrier)
            ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
            if (lane < KB) {
              const uint32_t* cnt = args.done + (n_blk * PARTS + i) * num_mp + lane;
              const uint32_t need = static_cast<uint32_t>(2 * (s + 1));
              while (dep::ld_acquire(cnt) < need) __nanosleep(32);
              dep::fence_proxy_async_global();
              if (lane == 0) stamp(g, s, i, 0);
              const uint32_t fb = ptx::mapa(fullk_bar(stage, lane), 0);
              ptx::mbar_arrive_expect_tx_cluster(fb, b_bytes);
              ptx::tma_load_2d_pair_hint(b_base + stage * Cfg::STAGE_BYTES + lane * b_bytes,
                                         &maps.g.Gin[Cfg::cls(i)][s & 1], fb, lane * Cfg::BK, b_row0, keep);
            }
            __syncwarp();
          } else {
            dep::wait_block(args.done, PARTS * n_blk + i, 0u, static_cast<uint32_t>((s + 1) * args.num_m));
            if (lane == 0) stamp(g, s, i, 0);
            ptx::mbar_wait(empty_bar(stage), ph ^ 1u);
            if (lane == 0) stamp(g, s, i, 8);
            if (ptx::elect_one()) {
              const uint32_t fb = ptx::mapa(full_bar(stage), 0);
              if constexpr (Cfg::KH2) {
                const int kh = KB / 2;
                const uint32_t fb2 = ptx::mapa(full2_bar(stage), 0);
                ptx::mbar_arrive_expect_tx_cluster(fb, kh * b_bytes);
                ptx::tma_load_3d_pair_hint(b_base + stage * Cfg::STAGE_BYTES, &maps.Gin3h[Cfg::cls(i)][s & 1], fb, 0,
                                           b_row0, 0, keep);
                ptx::mbar_arrive_expect_tx_cluster(fb2, kh * b_bytes);
                ptx::tma_load_3d_pair_hint(b_base + stage * Cfg::STAGE_BYTES + kh * b_bytes,
                                           &maps.Gin3h[Cfg::cls(i)][s & 1], fb2, 0, b_row0, kh, keep);
              } else {
                ptx::mbar_arrive_expect_tx_cluster(fb, KB * b_bytes);
                ptx::tma_load_3d_pair_hint(b_base + stage * Cfg::STAGE_BYTES, &maps.g.Gin3[Cfg::cls(i)][s & 1], fb,
                                           0, b_row0, 0, keep);
              }
            }
            __syncwarp();
          }
          if (++stage == STAGES) {
            stage = 0;
            ph ^= 1u;
          }
        });
      }
    }
  } else if (warp == 1) {  // ------------------------------------------ MMA issuer (leader)
    if (leader) {
      const uint32_t sf = tmem_base + Cfg::COL_SF;
      int stage = 0;
      uint32_t ph = 0;
      int lt = 0;
      for (int g = args.group0; g < args.group0 + args.groups; ++g) {
        const int n_blk = g * args.rb_per_group + rbk;
        if (n_blk >= num_n) break;
        for (int s = 0; s < args.nsteps; ++s, ++lt) {
          static_for<0, PARTS>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr uint32_t idesc = ptx::idesc_mxf4(256, Cfg::w(i));
            ptx::mbar_wait(tempty_bar(i), (lt & 1) ^ 1u);
            if constexpr (!Cfg::PKB) ptx::mbar_wait(full_bar(stage), ph);
            if (lane == 0) {
              stamp(g, s, i, 6);
              stamp(g, s, i, 7);
            }
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
              const uint32_t d = tmem_base + Cfg::off(i);
              const uint32_t bb = b_base + stage * Cfg::STAGE_BYTES;
              auto kblock = [&](int kb, bool first) {
                const uint64_t bdesc = ptx::smem_desc_k_sw128(bb + kb * (Cfg::w(i) / 2) * Cfg::BK);
                const uint32_t a = tmem_base + Cfg::COL_J + kb * 32;
#pragma unroll
                for (int k = 0; k < Cfg::BK / 32; ++k)
                  ptx::mma_mxf4_pair_ts(d, a + 8 * k, bdesc + 2 * k, idesc, sf, !(first && k == 0));
              };
              if constexpr (Cfg::PKB) {
                // K blocks in the order their slabs land; the first one issued zero-initialises
                uint32_t left = (1u << KB) - 1u;
                bool first = true;
                while (left) {
                  for (int kb = 0; kb < KB; ++kb)
                    if (((left >> kb) & 1u) && ptx::mbar_test_wait(fullk_bar(stage, kb), ph)) {
                      ptx::tc_fence_after();
                      kblock(kb, first);
                      first = false;
                      left &= ~(1u << kb);
                    }
                }
              } else if constexpr (Cfg::KH2) {
                for (int kb = 0; kb < KB / 2; ++kb) kblock(kb, kb == 0);
                ptx::mbar_wait(full2_bar(stage), ph);  // the second half of the part-step's G
                ptx::tc_fence_after();
                for (int kb = KB / 2; kb < KB; ++kb) kblock(kb, false);
              } else {
                for (int kb = 0; kb < KB; ++kb) kblock(kb, kb == 0);
              }
              ptx::mma_commit_pair_mc(empty_bar(stage), 0x3);
              ptx::mma_commit_pair_mc(tfull_bar(i), 0x3);
            }
            __syncwarp();
            if (lane == 0) stamp(g, s, i, 9);
            if (++stage == STAGES) {
              stage = 0;
              ph ^= 1u;
            }
          });
        }
      }
    }
  } else if (warp == 2) {  // ------------------------------------------ G_0 helper (later groups)
    // as in the parts kernel: publish group g's G_0 = sgn(x_0) from global x while group g - 1
    // steps, and prefetch g's state rows into L2 for its TMA loads
    const int64_t gpitch = args.npad / 2;
    const int gvalid = (args.n + 1) / 2;
    const int q = lane & 3;
    const int b0 = i0 / 2 + q * 16;
    for (int g = args.group0 + 1; g < args.group0 + args.groups; ++g) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      while (*started < g - args.group0) __nanosleep(256);
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
        dep::fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) dep::release_add(args.done + done_idx(n_blk, i), 1u);
      });
      if (lane == 0) gstamp(g, 6);
      for (int rr = lane; rr < Cfg::NR; rr += 32) {
        const int r = n_blk * Cfg::NR + rr;
        if (r >= args.rpad) break;
        const size_t off = static_cast<size_t>(r) * args.npad + i0;
        ptx::prefetch_l2_bulk(args.y + off, Cfg::BM * 4);
        ptx::prefetch_l2_bulk(args.p + off, Cfg::BM * 4);
        ptx::prefetch_l2_bulk(args.x + off, Cfg::BM * 4);
      }
    }
  } else if (warp == 3) {  // ------------------------------------------ G publisher
    // One thread publishes every part in turn (parts complete in order): TMA store of the part's
    // G tile, completion, proxy fence and red.release of its counter. (One lane per part, as in
    // the parts kernel, measured 28.6 vs 26.5 us/step: the four diverged lanes' waits serialise
    // inside the warp anyway and add latency; the release itself costs ~0.6 us either way.)
    if (lane == 0) {
      ptx::prefetch_tmap(&maps.g.Gout[0][0]);
      ptx::prefetch_tmap(&maps.g.Gout[0][1]);
      ptx::prefetch_tmap(&maps.g.Gout[1][0]);
      ptx::prefetch_tmap(&maps.g.Gout[1][1]);
      for (int c = 0; c < 2; ++c) {
        ptx::prefetch_tmap(&maps.X[c]);
        ptx::prefetch_tmap(&maps.Y[c]);
      }
      // x, y of a group's part k: one 2D TMA box each into shared memory (rows >= rpad
      // zero-filled), completing on sfull(k); the epilogue waits for it before the part's step 0
      auto load_state = [&](int g, int k_off, int k_cls, int k_w, int k) {
        const int n_blk = g * args.rb_per_group + rbk;
        if (args.ready)
          while (dep::ld_acquire_sys(args.ready + (g == 0 ? rbk : args.rb_per_group + g - 1)) == 0)
            __nanosleep(256);
        const uint32_t so = static_cast<uint32_t>(k_off * Cfg::BM * 4);
        ptx::mbar_arrive_expect_tx(sfull_bar(k), 2u * k_w * Cfg::BM * 4u);
        ptx::tma_load_2d(x_base + so, &maps.X[k_cls], sfull_bar(k), i0, n_blk * Cfg::NR + k_off);
        ptx::tma_load_2d(y_base + so, &maps.Y[k_cls], sfull_bar(k), i0, n_blk * Cfg::NR + k_off);
      };
      if (args.group0 * args.rb_per_group + rbk < num_n)
        static_for<0, PARTS>([&](auto I) {
          constexpr int k = decltype(I)::value;
          load_state(args.group0, Cfg::off(k), Cfg::cls(k), Cfg::w(k), k);
        });
      int pc = 0;
      for (int g = args.group0; g < args.group0 + args.groups; ++g) {
        const int n_blk = g * args.rb_per_group + rbk;
        if (n_blk >= num_n) break;
        const bool next = g + 1 < args.group0 + args.groups && (g + 1) * args.rb_per_group + rbk < num_n;
        // G_0 of the launch's first group (the epilogue writes it at group start), then G_{s+1}
        for (int s = g == args.group0 ? -1 : 0; s < args.nsteps; ++s, ++pc) {
          const int par = s < 0 ? 1 : (s & 1);
          static_for<0, PARTS>([&](auto I) {
            constexpr int k = decltype(I)::value;
            ptx::mbar_wait(gfull_bar(k), pc & 1);
            stamp(g, s, k, 3);
            ptx::tma_store_2d(&maps.g.Gout[Cfg::cls(k)][par], t_base + Cfg::off(k) * (Cfg::BM / 2), i0 / 2,
                              n_blk * Cfg::NR + Cfg::off(k));
            if (s == args.nsteps - 1) {
              // the group's last step: part k's x, y go back to global memory now (the
              // epilogue's smem writes were proxy-fenced before its gfull arrival), overlapping
              // the other parts' last step; gempty(k) below then also frees them for the next
              // group's loads
              const uint32_t so = static_cast<uint32_t>(Cfg::off(k) * Cfg::BM * 4);
              ptx::tma_store_2d(&maps.X[Cfg::cls(k)], x_base + so, i0, n_blk * Cfg::NR + Cfg::off(k));
              ptx::tma_store_2d(&maps.Y[Cfg::cls(k)], y_base + so, i0, n_blk * Cfg::NR + Cfg::off(k));
            }
            ptx::bulk_commit();
            ptx::bulk_wait_read0();
            // the group's last step: part k's buffers are free, the next group's part k loads now
            if (s == args.nsteps - 1 && next) load_state(g + 1, Cfg::off(k), Cfg::cls(k), Cfg::w(k), k);
            ptx::mbar_arrive(gempty_bar(k));  // tile reusable
            ptx::bulk_wait0();
            stamp(g, s, k, 4);
            // red.release orders the completed (proxy-fenced) tile writes before the count
            dep::fence_proxy_async_global();
            dep::release_add(args.done + done_idx(n_blk, k), 1u);
            stamp(g, s, k, 5);
            // dev skew trace (SBG_RES_GTRACE): every CTA's release time of part 0, steps 8..39 of group 0
            if (SBG_DEVHOOKS && k == 0 && SBG_HOOK_PTR(args.gtrace) && g == args.group0 && s >= 8 && s < 40) {
              uint32_t smid;
              asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
              SBG_HOOK_PTR(args.gtrace)[size_t(gridDim.x) * 512 + size_t(blockIdx.x) * 32 + (s - 8)] =
                  (gtimer() & 0xFFFFFFFFFFFFull) | (uint64_t(smid) << 48);
            }
          });
        }
      }
    }
#if SBG_TS_REGS
  }
  } else {
    ptx::setmaxnreg_inc<104>();
#else
  } else {  // ------------------------------------------------------------- epilogue
#endif
    const int q = warp & 3;
    const int cg = (warp - 4) >> 2;
    const int sl = q * 32 + lane;  // this thread's spin within the CTA
    const int spin = i0 + sl;
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t g_sel = (lane & 1) ? 0x15u : 0x40u;
    const bool io = warp == 4 && lane == 0;  // dev trace stamps, the helper pacing signal
    auto xa = [&](int col) { return x_base + static_cast<uint32_t>(col * Cfg::BM + sl) * 4u; };
    auto ya = [&](int col) { return y_base + static_cast<uint32_t>(col * Cfg::BM + sl) * 4u; };
    float preg[Cfg::NR / 4];
    // p of part I of replica block nb: this thread's spin, its column quarter of the part
    auto load_p = [&](auto I, int nb) {
      constexpr int i = decltype(I)::value;
      static_for<0, Cfg::w(i) / 16>([&](auto C) {
        constexpr int c = decltype(C)::value;
        const int col = Cfg::off(i) + cg * (Cfg::w(i) / 4) + c * CH;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = nb * Cfg::NR + col + j;
          preg[Cfg::off(i) / 4 + c * CH + j] = r < args.rpad ? args.p[static_cast<size_t>(r) * args.npad + spin] : 0.0f;
        }
      });
    };
    auto store_p = [&](auto I, int nb) {
      constexpr int i = decltype(I)::value;
      const uint64_t wb_policy = ptx::policy_evict_first();
      static_for<0, Cfg::w(i) / 16>([&](auto C) {
        constexpr int c = decltype(C)::value;
        const int col = Cfg::off(i) + cg * (Cfg::w(i) / 4) + c * CH;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int r = nb * Cfg::NR + col + j;
          if (r < args.rpad)
            ptx::st_hint(args.p + static_cast<size_t>(r) * args.npad + spin,
                         __float_as_uint(preg[Cfg::off(i) / 4 + c * CH + j]), wb_policy);
        }
      });
    };
    auto put_g2 = [&](int row, float xa_, float xb_) {
      const uint32_t mine = (xa_ >= 0.0f ? 0x2u : 0xAu) | ((xb_ >= 0.0f ? 0x2u : 0xAu) << 8);
      const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, mine, 1);
      const uint32_t t = __byte_perm(mine, other, g_sel);
      g_tile[(row + (lane & 1)) * (Cfg::BM / 2) + (sl >> 1)] = static_cast<uint8_t>(t | (t >> 4));
    };
    auto tile_written = [&](int i) {
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(gfull_bar(i));
    };
    int lt = 0, pc = 0, gl = 0;
    for (int g = args.group0; g < args.group0 + args.groups; ++g, ++gl) {
      const int n_blk = g * args.rb_per_group + rbk;
      if (n_blk >= num_n) break;
      const bool first = g == args.group0;
      if (io) gstamp(g, 0);
      // ---- group start: x, y arrive by TMA (issued by the publisher, sfull), p to registers
      // (SBG_TS_PPART: later groups' p was loaded part by part during the previous group's last step)
      if (first || !SBG_TS_PPART)
        static_for<0, PARTS>([&](auto I) { load_p(I, n_blk); });
      if (first) {  // G_0 = sgn(x_0) of the launch's first group (later groups: the helper)
        static_for<0, PARTS>([&](auto I) {
          constexpr int i = decltype(I)::value;
          ptx::mbar_wait(gempty_bar(i), (pc & 1) ^ 1u);
          ptx::mbar_wait(sfull_bar(i), gl & 1);
          static_for<0, Cfg::w(i) / 16>([&](auto C) {
            constexpr int c = decltype(C)::value;
            const int col = Cfg::off(i) + cg * (Cfg::w(i) / 4) + c * CH;
            put_g2(col, ptx::lds_f32(xa(col)), ptx::lds_f32(xa(col + 1)));
            put_g2(col + 2, ptx::lds_f32(xa(col + 2)), ptx::lds_f32(xa(col + 3)));
          });
          tile_written(i);
        });
        ++pc;
      }
      if (io) {
        *started = g - args.group0 + 1;
        gstamp(g, 1);
      }
      for (int s = 0; s < args.nsteps; ++s, ++lt, ++pc) {
        PhaseConsts k = args.k;
        k.inv = __frcp_rn(static_cast<float>(args.M - (args.t_begin + static_cast<uint64_t>(s))));
        const PhaseConsts2 k2(k, args.ident);
        const float* arep = args.a_rep;
        static_for<0, PARTS>([&](auto I) {
          constexpr int i = decltype(I)::value;
          constexpr int CHUNKS = Cfg::w(i) / 16;
          const int c0 = Cfg::off(i) + cg * (Cfg::w(i) / 4);
          float bx[2][CH], by[2][CH];
          auto ld_xy = [&](int c, int b) {
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              bx[b][j] = ptx::lds_f32(xa(c0 + c * CH + j));
              by[b][j] = ptx::lds_f32(ya(c0 + c * CH + j));
            }
          };
          if (s == 0) ptx::mbar_wait(sfull_bar(i), gl & 1);  // this part's state has landed
          ld_xy(0, 0);  // the state does not depend on the MMA: read before its completion
          ptx::mbar_wait(tfull_bar(i), lt & 1);
          __syncwarp();
          ptx::tc_fence_after();
          if (io && i == 0 && s < 2) gstamp(g, 2 + s);
          if (io) stamp(g, s, i, 1);
#if SBG_TS_LD1
          // this warp's whole slice of the part's field (W/4 columns) in one or two tcgen05.ld
          // and ONE wait: the per-chunk load-wait round trips (~0.2 us each under the MMAs'
          // TMEM traffic) were most of the epilogue's time
          constexpr int NC = Cfg::w(i) / 4;
          uint32_t fv[NC];
          if constexpr (NC == 12) {
            ptx::tmem_ld<8>(t_lane + c0, *reinterpret_cast<uint32_t(*)[8]>(&fv[0]));
            ptx::tmem_ld<4>(t_lane + c0 + 8, *reinterpret_cast<uint32_t(*)[4]>(&fv[8]));
          } else if constexpr (NC == 8) {
            ptx::tmem_ld<8>(t_lane + c0, *reinterpret_cast<uint32_t(*)[8]>(&fv[0]));
          } else {
            static_assert(NC == 8 || NC == 12, "part widths 48 / 32");
          }
          ptx::mbar_wait(gempty_bar(i), (pc & 1) ^ 1u);  // this part's G tile stored (under the load)
          if (io) stamp(g, s, i, 10);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < NC; ++j) asm volatile("" : "+r"(fv[j]));
          if (io) stamp(g, s, i, 11);
          auto fld = [&](int c, int j) { return __uint_as_float(fv[c * CH + j]); };
#else
          uint32_t bf[2][CH];
          ptx::tmem_ld<CH>(t_lane + c0, bf[0]);
          ptx::mbar_wait(gempty_bar(i), (pc & 1) ^ 1u);  // this part's G tile stored (under the load)
          if (io) stamp(g, s, i, 10);
          ptx::tmem_ld_wait();
          if (io) stamp(g, s, i, 11);
          auto fld = [&](int c, int j) { return __uint_as_float(bf[c & 1][j]); };
#endif
          auto chunks = [&](auto has_arep) {
            static_for<0, CHUNKS>([&](auto C) {
              constexpr int c = decltype(C)::value;
              constexpr int b = c & 1;
              if constexpr (c + 1 < CHUNKS) {
#if !SBG_TS_LD1
                ptx::tmem_ld<CH>(t_lane + c0 + (c + 1) * CH, bf[b ^ 1]);
#endif
                ld_xy(c + 1, b ^ 1);
              }
              const int col = c0 + c * CH;
#pragma unroll
              for (int j = 0; j < CH; j += 2) {
                float x0 = bx[b][j], x1 = bx[b][j + 1];
                float y0 = by[b][j], y1 = by[b][j + 1];
                float& p0 = preg[Cfg::off(i) / 4 + c * CH + j];
                float& p1 = preg[Cfg::off(i) / 4 + c * CH + j + 1];
                uint64_t a2 = k2.a;
                if constexpr (decltype(has_arep)::value) {
                  const int r = n_blk * Cfg::NR + col + j;
                  a2 = f2::pk(arep[min(r, args.R - 1)], arep[min(r + 1, args.R - 1)]);
                }
                gsb_phase2(fld(c, j), fld(c, j + 1), x0, x1, y0, y1, p0, p1, k2, a2);
                ptx::sts_f32(xa(col + j), x0);
                ptx::sts_f32(xa(col + j + 1), x1);
                ptx::sts_f32(ya(col + j), y0);
                ptx::sts_f32(ya(col + j + 1), y1);
                put_g2(col + j, x0, x1);
              }
#if !SBG_TS_LD1
              if constexpr (c + 1 < CHUNKS) {
                ptx::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < CH; ++j) asm volatile("" : "+r"(bf[b ^ 1][j]));
              }
#endif
            });
          };
          if (arep)
            chunks(std::true_type{});
          else
            chunks(std::false_type{});
          if (io) stamp(g, s, i, 12);
          tile_written(i);
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(ptx::mapa(tempty_bar(i), 0));
          if (io) stamp(g, s, i, 2);
          if constexpr (SBG_TS_PPART) {
            // the group's last step: this part's p goes back now and the next group's p of this
            // part is loaded into the same registers (consumed at its step 0), overlapping the
            // other parts' last-step epilogues
            if (s == args.nsteps - 1) {
              store_p(I, n_blk);
              const int nb = (g + 1) * args.rb_per_group + rbk;
              if (g + 1 < args.group0 + args.groups && nb < num_n) load_p(I, nb);
            }
          }
        });
      }
      // ---- group end: x, y went back with the last step's G tiles (the publisher); p by stores
      if (io) gstamp(g, 4);
      if (!SBG_TS_PPART) static_for<0, PARTS>([&](auto I) { store_p(I, n_blk); });
      if (io) gstamp(g, 5);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, 512);
}

}  // namespace sbg
