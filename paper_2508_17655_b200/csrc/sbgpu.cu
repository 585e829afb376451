// sbgpu context and C ABI (include/sbgpu.h).
//
// Owns the device copies of J, the replica states, the B-operand planes and
// the TMA descriptors; drives the per-step tensor-core kernel (step_i8.cuh)
// M times, then the readout. Replaces, for this path, sbopt::run's loop
// (/root/reference/proj/core/src/engine.cpp:112-139) fanned out over replicas
// by the reference's ThreadPool (bench.cpp:70-92, parallel.cpp:59-84).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/sbgpu.h"
#include "aux_kernels.cuh"
#include "e2m1.cuh"
#include "csr_step.cuh"
#include "gen_dense.cuh"
#include "spectral.cuh"
#include "step_i8.cuh"
#include "step_tma.cuh"
#include "step_pair.cuh"
#include "step_resident.cuh"
#include "step_resident_parts.cuh"
#include "step_resident_ts.cuh"

using namespace sbg;

namespace {

constexpr int BN_SIGN = 128;   // replica tile, sign variants (dsb/gdsb)
constexpr int BN_PLANE = 64;   // replica tile, fixed-point variants (bsb/gbsb)
constexpr int NPL = 4;         // fixed-point byte planes
constexpr int PAD_N = 256;     // spin padding (pair MMA M = 256, K granularity 128)
constexpr int PAD_R = 256;     // replica padding (multiple of every replica tile)
constexpr int NPAIR_SIGN = 256;   // replicas per pair tile, sign variants
constexpr int NPAIR_PLANE = 64;   // replicas per pair tile, fixed-point variants

enum Kind { KIND_NONE = 0, KIND_DENSE_I8 = 1, KIND_CSR_I8 = 2, KIND_DENSE_FX = 3 };
constexpr int FX_NA = 3;          // real J: 24-bit fixed point as 3 byte planes (u8, u8, s8)
constexpr int BN_FX_SIGN = 64;    // replica tile, real J x sign plane (3 accumulators)
constexpr int BN_FX_PLANE = 32;   // replica tile, real J x 4 x-planes (6 accumulators, double-buffered)
constexpr int BN_FX_PLANE_W = 64; // the same with one accumulator buffer (default; == BN_PLANE)
static_assert(BN_FX_PLANE_W == BN_PLANE, "the 64-wide real-J launch uses the maps_planes G boxes");

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool is_sign_variant(int v) { return v == SBG_DSB || v == SBG_GDSB; }

using PFN_writeValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_writeValue32 get_write_value32() {
  static PFN_writeValue32 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_writeValue32>(p);
  }
  return fn;
}

}  // namespace

// Tensor maps of the TS kernel for one G-buffer parity, valid while this key holds (the
// launch then does no host-side encoding: the timed advance's GPU idle time before the
// kernel is only the launch itself).
struct TsMapKey {
  const void *g0 = nullptr, *g1 = nullptr, *x = nullptr, *y = nullptr, *j4 = nullptr;
  int64_t n = 0, npad = 0, R = 0, rpad = 0;
  int w0 = 0, w1 = 0;
  bool operator==(const TsMapKey& o) const {
    return g0 == o.g0 && g1 == o.g1 && x == o.x && y == o.y && j4 == o.j4 && n == o.n && npad == o.npad && R == o.R &&
           rpad == o.rpad && w0 == o.w0 && w1 == o.w1;
  }
};

struct sbg_ctx {
  int device = 0;
  TsMaps ts_cache[2];
  void* d_fused = nullptr;  // sbg_shard_advance_fused: rank tables (maps, args)
  size_t fused_cap = 0;
  TsMapKey ts_key[2];
  bool ts_ok[2] = {false, false};
  int sms = 148;
  std::string device_name;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;
  // couplings
  int kind = KIND_NONE;
  int64_t n = 0, npad = 0;
  int8_t* dJ = nullptr;
  CUtensorMap tmJ;
  // packed e2m1 copy of an e2m1-exact dense int8 J ([npad][npad / 2]; e2m1.cuh): the sign
  // variants' resident kernel then runs kind::mxf4 MMAs (SBG_Q4=0 disables, dev)
  uint8_t* dJ4 = nullptr;
  CUtensorMap tmJ4;
  CUtensorMap tmJplane[FX_NA];  // KIND_DENSE_FX: one map per J byte plane (readout)
  int fx_shift = 0;             // KIND_DENSE_FX: J_int = rint(J * 2^fx_shift)
  double energy_scale = 1.0;    // energy = -E2/2 * energy_scale (2^-fx_shift for real J)
  int32_t* d_rowptr = nullptr;
  int32_t* d_col = nullptr;
  int8_t* d_val = nullptr;
  int64_t nnz = 0;
  // replica state
  int64_t R = 0, rpad = 0, cap_rpad = 0;
  float *dX = nullptr, *dY = nullptr, *dP = nullptr;
  uint8_t* dG[2] = {nullptr, nullptr};  // B-operand buffers, NPL planes each
  uint8_t* dSign = nullptr;             // readout sign plane
  int8_t* dSignAll = nullptr;           // row shard readout: private byte plane of all spins'
  size_t sign_all_bytes = 0;            // signs (peers never write it), [rpad][kpad]
  CUtensorMap tmSignAll;
  unsigned long long* dE2 = nullptr;
  long long* dBest = nullptr;
  CUtensorMap tmG_sign[2], tmG_planes[2], tmSign;
  TmaMaps maps_sign[2], maps_planes[2];  // multi-step kernel maps, indexed by the current B buffer
  TmaMaps pmaps_planes[2];               // pair kernel, fixed-point planes (B half = 32 rows)
  TmaMaps fxmaps_sign[2], fxmaps_planes[2];  // real-J kernels (B tiles of 64 / 32 rows)
  // real J x 4 digit planes: 64-byte K stages (TmaStepCfg::BK = 64, 64-byte swizzle), B tiles
  // of 64 / 32 replica rows; J (tmJfx64) is set at launch
  TmaMaps fxq_planes64[2], fxq_planes32[2];
  CUtensorMap tmJfx64;
  TmaMaps maps_sign_cw8[2];                  // sign pair kernel with 8-replica state chunks
  TmaMaps rmaps_sign[2];                     // resident-state pair kernel, NR 128 (B halves of 64 rows)
  TmaMaps rmaps160_sign[2];                  // resident-state pair kernel, NR 160 (B halves of 80 rows)
  TmaMaps qmaps_sign[2], qmaps160_sign[2];   // the same on e2m1 operands (J4; G as [rpad][npad / 2])
  TmaMaps pqmaps_sign[2];                    // streaming sign pair kernel on e2m1 operands
  TmaMaps pq128maps_sign[2];                 // the same with 128-replica pair tiles
  unsigned long long* dE2p = nullptr;    // real-J readout: per-J-plane partial E2 [FX_NA][rpad]
  // CSR: spin-major working copies [npad][rp] and the ping-pong gathered operand (q int32 / sign int8)
  float *dXs = nullptr, *dYs = nullptr, *dPs = nullptr;
  int32_t* dQ[2] = {nullptr, nullptr};
  int64_t rp = 0;
  // Row sharding (C5): this context owns spins [row0, row0 + npad) of an n_global problem;
  // the contraction runs over kpad = padded n_global columns. Unsharded: n_global = n, row0 = 0.
  bool sharded = false;
  int64_t n_global = 0, kpad = 0, row0 = 0, num_m_total = 0;
  uint32_t done_base = 0;  // done[] counters run on across launches (peers increment them)
  std::vector<uint8_t*> peer_g0, peer_g1;
  std::vector<uint32_t*> peer_done;
  uint32_t* d_err = nullptr;  // row shards: peer-wait timeout flag (MultiStepArgs::err)
  float* d_fpart = nullptr;  // K-split partial fields (pair kernel), fpart_cap floats
  size_t fpart_cap = 0;
  uint32_t* d_kdone = nullptr;
  size_t kdone_cap = 0;
  float* d_arep = nullptr;  // optional per-replica A (sbg_set_replica_a), honoured by gbsb/gdsb
  int64_t arep_n = 0;
  uint32_t* d_done = nullptr;            // per replica-block tile counters of the multi-step kernel
  uint32_t* d_ready = nullptr;           // per replica-group "state copied" flags (sbg_run pipelining)
  int64_t ready_cap = 0;
  int g_cur = 0;
  int g_mode = 0;  // 0 stale, 1 sign plane valid in dG[g_cur], 2 e2m1 sign plane, 4 planes valid
  cudaEvent_t ev[8];
  cudaStream_t cstream = nullptr;  // host->device copies overlapped with the resident kernel (sbg_run)
  cudaEvent_t evc[3];
  float last_advance_ms = 0.f;
  int8_t* tail_best_spins = nullptr;  // sbg_run_best: winner-only readout in run_tail
  bool csr_sm_current = false;  // CSR: the spin-major working copies hold the state (dX/dY/dP stale)
  int csr_q = -1;               // ... and dQ[csr_q] holds its gathered operand (sign: +2), -1 none
  double* tail_best_energy = nullptr;

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
};

// Width (bytes per replica row) of the B-operand buffers: all spins of the problem.
int64_t gdim(const sbg_ctx* ctx) { return ctx->sharded ? ctx->kpad : ctx->npad; }

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return ctx->fail(e_ == cudaErrorMemoryAllocation ? SBG_ERR_OUT_OF_MEMORY : SBG_ERR_CUDA, \
                       "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define CHECK_CTX(ctx) \
  if (!(ctx)) return SBG_ERR_INVALID_ARGUMENT

// Row shards: a peer wait that timed out on the device (MultiStepArgs::err) is an error.
static int shard_wait_check(sbg_ctx* ctx) {
  if (!ctx->sharded || !ctx->d_err) return SBG_OK;
  uint32_t e = 0;
  CK(cudaMemcpy(&e, ctx->d_err, sizeof e, cudaMemcpyDeviceToHost));
  if (e) return ctx->fail(SBG_ERR_CUDA, "row shard: a peer rank did not release its slab within 4 s "
                                        "(peer died, not launched, or not wired); results are invalid");
  return SBG_OK;
}


namespace {

int encode_2d_u8(sbg_ctx* ctx, CUtensorMap* tm, const void* base, uint64_t inner, uint64_t rows,
                 uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto enc = get_encode();
  if (!enc) return ctx->fail(SBG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return ctx->fail(SBG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return SBG_OK;
}

int encode_2d(sbg_ctx* ctx, CUtensorMap* tm, CUtensorMapDataType dt, uint32_t esize, const void* base,
              uint64_t inner, uint64_t rows, uint64_t row_pitch_bytes, uint32_t box_inner, uint32_t box_rows,
              CUtensorMapSwizzle swz) {
  auto enc = get_encode();
  if (!enc) return ctx->fail(SBG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_pitch_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  (void)esize;
  CUresult r = enc(tm, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return ctx->fail(SBG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  return SBG_OK;
}

int grid_for(const sbg_ctx* ctx, size_t work, int threads) {
  const size_t blocks = (work + threads - 1) / threads;
  return static_cast<int>(std::min<size_t>(std::max<size_t>(blocks, 1), size_t(ctx->sms) * 8));
}

template <int NP, int BN, EpiMode MODE>
int launch_step(sbg_ctx* ctx, const CUtensorMap& tmG, const StepArgs& a, const CUtensorMap* tmA = nullptr) {
  using Cfg = StepCfg<NP, BN>;
  auto kern = gsb_step_i8_kernel<NP, BN, MODE>;
  static int attr_device = -1;  // once per instantiation and device
  if (attr_device != ctx->device) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_device = ctx->device;
  }
  const int tiles = a.num_m * a.num_n;
  const int grid = std::min(tiles, ctx->sms);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, ctx->stream>>>(tmA ? *tmA : ctx->tmJ, tmG, a);
  CK(cudaGetLastError());
  ++ctx->launches;
  return SBG_OK;
}

// Multi-step persistent launch (step_tma.cuh). Sign variants: BN 128, 4 operand
// stages, 3 state buffers; fixed-point planes: BN 64, 3 stages, 2 buffers
// (best of the measured (stages, buffers) sweeps on B200).
constexpr int SIGN_STAGES = 4, SIGN_NBUF = 3;
constexpr int PLANE_STAGES = 3, PLANE_NBUF = 2;

int dev_knob(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}
// Knobs that need the dev hooks compiled into the kernels (SBG_DEVHOOKS, `build.py --devhooks`):
// in the shipped library they are refused loudly instead of silently tracing nothing.
int hook_knob(const char* name) {
  const int v = dev_knob(name);
  if (v && !SBG_DEVHOOKS) {
    static bool warned = false;
    if (!warned)
      fprintf(stderr, "sbgpu: %s ignored: this library was built without dev hooks "
                      "(python paper_2508_17655_b200/build.py --devhooks builds libsbgpu_dev.so)\n", name);
    warned = true;
    return 0;
  }
  return v;
}
bool getenv_is0(const char* name) {
  const char* e = getenv(name);
  return e && atoi(e) == 0;
}

// Persistent multi-step kernels spin on counters released by other CTAs of the
// same launch, so every CTA must be resident at once: launch them cooperatively
// (the driver then never co-schedules them partially next to another kernel).
template <typename... KArgs, typename... Args>
cudaError_t launch_persistent(void (*kern)(KArgs...), int grid, int block, int smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(block));
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <int NP, int BN, int ST, int NB, int NA = 1>
int launch_multistep(sbg_ctx* ctx, const TmaMaps& maps, const MultiStepArgs& a) {
  using Cfg = TmaStepCfg<NP, BN, ST, NB, NA>;
  auto kern = gsb_multistep_kernel<NP, BN, ST, NB, NA>;
  static int attr_device = -1;  // once per instantiation and device
  if (attr_device != ctx->device) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_device = ctx->device;
  }
  const int64_t tiles = int64_t(a.num_m) * a.num_n * a.nsteps;
  // persistent: one CTA per SM (all must be co-resident for the dependency walk)
  const int grid = int(std::min<int64_t>(tiles, ctx->sms));
  if (!ctx->sharded) CK(cudaMemsetAsync(ctx->d_done, 0, sizeof(uint32_t) * a.num_n, ctx->stream));
  CK(launch_persistent(kern, grid, Cfg::THREADS, Cfg::SMEM_BYTES, ctx->stream, maps, a));
  ++ctx->launches;
  if (ctx->sharded) ctx->done_base += uint32_t(a.nsteps * a.num_m_total);
  return SBG_OK;
}

template <int NP, int NPAIR, int ST, int NB, int CW = 16, bool Q4 = false, int NA = 1>
int launch_multistep_pair(sbg_ctx* ctx, const TmaMaps& maps, MultiStepArgs a) {
  using Cfg = PairStepCfg<NP, NPAIR, ST, NB, CW, Q4, NA>;
  auto kern = gsb_multistep_pair_kernel<NP, NPAIR, ST, NB, CW, Q4, NA>;
  static int attr_device = -1;  // once per instantiation and device
  if (attr_device != ctx->device) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_device = ctx->device;
  }
  a.num_n = int32_t(ctx->rpad / NPAIR);
  if (NP != 1) a.ksplit = 1;
  // every K part needs at least one K block: a part with an empty range would commit an
  // accumulator no MMA wrote (the previous tile's field)
  a.ksplit = std::min<int32_t>(a.ksplit, int32_t(a.kpad / (Cfg::BK * Cfg::KPB)));
  if (a.ksplit > 1) {
    const size_t need = size_t(a.ksplit - 1) * size_t(ctx->rpad) * size_t(ctx->npad);
    if (ctx->fpart_cap < need) {
      cudaFree(ctx->d_fpart);
      ctx->d_fpart = nullptr;
      ctx->fpart_cap = 0;
      CK(cudaMalloc(&ctx->d_fpart, sizeof(float) * need));
      ctx->fpart_cap = need;
    }
    const size_t nk = size_t(a.num_n) * size_t(a.num_m);
    if (ctx->kdone_cap < nk) {
      cudaFree(ctx->d_kdone);
      ctx->d_kdone = nullptr;
      ctx->kdone_cap = 0;
      CK(cudaMalloc(&ctx->d_kdone, sizeof(uint32_t) * nk));
      ctx->kdone_cap = nk;
    }
    CK(cudaMemsetAsync(ctx->d_kdone, 0, sizeof(uint32_t) * nk, ctx->stream));
    a.fpart = ctx->d_fpart;
    a.kdone = ctx->d_kdone;
  }
  const int64_t t2 = int64_t(a.num_m / 2) * a.num_n;
  const int64_t tt = a.ksplit > 1 ? (a.ktail > 0 ? std::min<int64_t>(a.ktail, t2) : t2) : 0;
  const int64_t pair_tiles = (t2 - tt + tt * std::max(1, a.ksplit)) * a.nsteps;  // work units
  const int grid = 2 * int(std::min<int64_t>(pair_tiles, ctx->sms / 2));
  if (!ctx->sharded) CK(cudaMemsetAsync(ctx->d_done, 0, sizeof(uint32_t) * a.num_n, ctx->stream));
  static unsigned long long* utrace = nullptr;  // dev knob SBG_PAIR_TRACE: per (CTA, unit) stamps
  const size_t utn = size_t(grid) * 64 * 8;
  if (hook_knob("SBG_PAIR_TRACE")) {
    cudaFree(utrace);
    CK(cudaMalloc(&utrace, utn * 8));
    CK(cudaMemsetAsync(utrace, 0, utn * 8, ctx->stream));
    a.utrace = utrace;
  }
  CK(launch_persistent(kern, grid, Cfg::THREADS, Cfg::SMEM_BYTES, ctx->stream, maps, a));
  ++ctx->launches;
  if (ctx->sharded) ctx->done_base += uint32_t(a.nsteps * a.num_m_total);
  if (a.utrace) {
    std::vector<unsigned long long> h(utn);
    CK(cudaMemcpyAsync(h.data(), a.utrace, utn * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    FILE* f = fopen("gpurun_out/pair_utrace.txt", "w");
    if (f) {
      for (size_t i = 0; i < utn / 8; ++i)
        if (h[i * 8 + 6] || h[i * 8])
          fprintf(f, "%zu %zu %llu %llu %llu %llu %llu %llu %llu\n", i / 64, i % 64, h[i * 8], h[i * 8 + 1],
                  h[i * 8 + 2], h[i * 8 + 3], h[i * 8 + 4], h[i * 8 + 5], h[i * 8 + 6]);
      fclose(f);
    }
  }
  return SBG_OK;
}

// K parts per pair tile (SBG_KSPLIT = n forces n parts; default 1). Splitting a tile's K range
// over several CTA pairs would fill the pairs a whole-tile schedule leaves idle in its last wave
// (C5: 49 tiles per rank at G = 8 on 74 pairs), and it is bitwise exact, but measured slower:
// G = 8 per-rank step 202 -> 257 us with 3 parts, single-GPU C5 1033 -> 1678 us (ncu: tensor
// pipe 61 -> 44 % of active cycles; the single accumulator buffer idles the MMAs while each
// part's partial field drains through global memory, and the last part waits on the others).
int ksplit_for(const sbg_ctx* ctx, int64_t tiles) {
  (void)ctx;
  (void)tiles;
  const int knob = dev_knob("SBG_KSPLIT");
  return knob > 1 ? std::min(knob, 8) : 1;
}

// Tail-only K split (default for the e2m1 streaming pair kernel; SBG_KTAIL=0 disables): with
// T2 pair tiles per step on P pairs and T2 >= P, the T2 mod P tiles of the last, partial round
// run as KS = min(4, P / (T2 mod P)) K parts each, so that round takes ~1/KS of a tile instead
// of a whole tile while every other pair idles (C5: 391 tiles on 74 pairs = 5 whole rounds + 21
// tiles). Sets a.ksplit / a.ktail; the explicit uniform split (SBG_KSPLIT) wins when set.
void tail_split(const sbg_ctx* ctx, int64_t tiles, MultiStepArgs& a) {
  a.ktail = 0;
  a.ksplit = ksplit_for(ctx, tiles);
  if (a.ksplit > 1 || getenv_is0("SBG_KTAIL")) return;
  const int64_t P = ctx->sms / 2, tail = tiles % P;
  if (tiles < P || tail == 0) return;
  const int64_t ks = std::min<int64_t>(4, P / tail);
  if (ks < 2) return;
  a.ksplit = int32_t(ks);
  a.ktail = int32_t(tail);
}

// 128-replica pair tiles, replica blocks fastest (SBG_Q4_NPAIR=128; default 256): meant to fill
// the pairs 256-replica tiles leave idle in the last wave while the replica blocks of one
// pair-block share its J reads in L2. Bitwise equal, measured slower (C5 single GPU 1045 ->
// 1277 us, G = 4 per rank 349 -> 364, G = 8 202 -> 264): half-width MMAs (N = 128) and twice the
// per-tile fixed costs outweigh the better wave fill.
bool q4_narrow(const sbg_ctx* ctx) {
  (void)ctx;
  return dev_knob("SBG_Q4_NPAIR") == 128;
}

// Sign variants streaming J on e2m1 operands (CTA pairs, kind::mxf4): the large-N regime
// (C5), row shards included; G is then the packed [rpad][kpad / 2] plane (g_mode 2).
bool q4_stream(const sbg_ctx* ctx) {
  return ctx->dJ4 && ctx->kind == KIND_DENSE_I8 && ctx->npad % 256 == 0 && dev_knob("SBG_STEP_CFG") == 0;
}

// Resident-state pair kernel (step_resident.cuh): sign variants, dense int8 J.
constexpr int RES_STAGES = 8;

bool resident_ok(const sbg_ctx* ctx);
bool use_resident(const sbg_ctx* ctx, int variant) {
  // default for sign variants on dense int8 J; SBG_RESIDENT=0 selects the streaming kernels (dev)
  return (variant == SBG_DSB || variant == SBG_GDSB) && !getenv_is0("SBG_RESIDENT") && resident_ok(ctx);
}

bool resident_ok(const sbg_ctx* ctx) {
  const int64_t num_mp = ctx->npad / 256;
  return ctx->kind == KIND_DENSE_I8 && !ctx->sharded && ctx->npad % 256 == 0 && num_mp >= 1 &&
         num_mp <= ctx->sms / 2;
}

// Replica-group geometry of the resident kernel: 128-replica blocks, num_mp pairs per block,
// as many blocks per group as CTA pairs fit (one CTA per SM).
constexpr int RES_NR = 160;  // replicas per pair block of the default resident kernel (p in smem)
constexpr int RES_NR_STAGES = 5;  // 32 of the 160 p columns stay in TMEM: room for a 5th ring stage

void resident_geometry(const sbg_ctx* ctx, int64_t npad, int64_t rpad, int* rb_per_group, int* groups,
                       int nr = RES_NR) {
  const int num_mp = int(npad / 256), num_n = int((rpad + nr - 1) / nr);
  *rb_per_group = std::min(num_n, (ctx->sms / 2) / num_mp);
  *groups = (num_n + *rb_per_group - 1) / *rb_per_group;
}

// NR 160 (p in shared memory) only pays when it cuts the number of sequential replica
// groups (C2: 8 -> 6); otherwise NR 128 is faster per group.
int resident_nr(const sbg_ctx* ctx) {
  int rb = 0, g128 = 0, g160 = 0;
  resident_geometry(ctx, ctx->npad, ctx->rpad, &rb, &g128, 128);
  resident_geometry(ctx, ctx->npad, ctx->rpad, &rb, &g160, RES_NR);
  // The TS kernel (e2m1 J in TMEM, npad <= 2048, four interleaved part chains) steps a 160-replica
  // block in ~4.6 us against ~6.2 us for a 128-replica block of the single-chain kernel: take it
  // whenever it does not ADD groups (R = 1000: 7 blocks of 160 instead of 8 of 128, one group either
  // way). SBG_RES_NR_TS=0 restores the group-count rule (dev A/B).
  const bool ts = ctx->dJ4 && !ctx->sharded && ctx->npad <= 2048 && !getenv_is0("SBG_RES_SPLIT") &&
                  !getenv_is0("SBG_RES_TS") && !getenv_is0("SBG_RES_NR_TS");
  if (ts && g160 <= g128) return RES_NR;
  return g160 < g128 ? RES_NR : 128;
}

template <int EPI, int CH, int ST = RES_STAGES, int NR = 128, bool Q4 = false, int PARTS = 0, bool JRES = false,
          class Maps = TmaMaps, bool PKB = false, bool KH2 = false>
int launch_resident(sbg_ctx* ctx, const Maps& maps, const MultiStepArgs& ms, int group0 = 0, int ngroups = -1,
                    const uint32_t* ready = nullptr) {
  // PARTS > 0: step_resident_parts.cuh (e2m1, 160-replica blocks as PARTS interleaved column
  // parts; JRES = J resident in shared memory); else step_resident.cuh
  // PARTS < 0: step_resident_ts.cuh with -PARTS parts (J in TMEM, x, y in shared memory)
  using Cfg = std::conditional_t<
      (PARTS < 0), TsCfg<ST, (PARTS < 0 ? -PARTS : 2), PKB, KH2>,
      std::conditional_t<(PARTS > 0), PartsCfg<ST, JRES, (PARTS > 0 ? PARTS : 2)>, ResCfg<ST, EPI, CH, NR, false, Q4>>>;
  auto kern = [] {
    if constexpr (PARTS < 0)
      return gsb_resident_ts_kernel<ST, -PARTS, PKB, KH2>;
    else if constexpr (PARTS > 0)
      return gsb_resident_parts_kernel<ST, JRES, PARTS>;
    else
      return gsb_resident_pair_kernel<ST, EPI, CH, NR, Q4>;
  }();
  static int attr_device = -1;  // once per instantiation and device (host work before the launch)
  if (attr_device != ctx->device) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_device = ctx->device;
  }
  ResidentArgs a;
  std::memset(&a, 0, sizeof a);
  a.n = ms.n;
  a.npad = ms.npad;
  a.R = ms.R;
  a.rpad = ms.rpad;
  a.num_m = ms.npad / Cfg::BM;
  const int num_mp = ms.npad / 256, num_n = (ms.rpad + Cfg::NR - 1) / Cfg::NR;
  int total_groups = 0;
  resident_geometry(ctx, ms.npad, ms.rpad, &a.rb_per_group, &total_groups, Cfg::NR);
  a.group0 = group0;
  a.groups = ngroups < 0 ? total_groups - group0 : ngroups;
  a.k = ms.k;
  a.M = ms.M;
  a.t_begin = ms.t_begin;
  a.nsteps = ms.nsteps;
  a.done = ctx->d_done;
  a.x = ctx->dX;
  a.y = ctx->dY;
  a.p = ctx->dP;
  a.a_rep = ms.a_rep;
  a.ident = PhaseIdent{-0.0f, 1.0f, -1.0f};
  a.ready = ready;
  a.gbuf[0] = ctx->dG[ctx->g_cur ^ 1];  // step parity 0 writes the other buffer (as Gout[0])
  a.gbuf[1] = ctx->dG[ctx->g_cur];
  a.dbg = hook_knob("SBG_STEP_DBG");
  a.j4 = ctx->dJ4;
  a.j4_pitch = ctx->npad / 2;
  static unsigned long long* trace = nullptr;  // dev knob SBG_RES_TRACE: stamps of pair 0, group 0
  if (hook_knob("SBG_RES_TRACE")) {
    if (!trace) CK(cudaMalloc(&trace, sizeof(unsigned long long) * 16 * 4 * 4096));
    CK(cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * 16 * 4 * 4096, ctx->stream));
    a.trace = trace;
    a.trace_group = hook_knob("SBG_RES_TRACE") - 1;  // 1 = the launch's first group, 2 = the second, ...
    a.nsteps = std::min(a.nsteps, 4096);
  }
  static unsigned long long* gtrace = nullptr;  // dev knob SBG_RES_GTRACE: per-(CTA, group) stamps
  const size_t gtn = size_t(ctx->sms) * 64 * 8 + size_t(ctx->sms) * 32;  // + the TS kernel's skew trace
  if (PARTS != 0 && hook_knob("SBG_RES_GTRACE")) {  // parts and TS kernels
    if (!gtrace) CK(cudaMalloc(&gtrace, sizeof(unsigned long long) * gtn));
    CK(cudaMemsetAsync(gtrace, 0, sizeof(unsigned long long) * gtn, ctx->stream));
    a.gtrace = gtrace;
  }
  // done counters per replica block (one per part)
  const int counters = PARTS != 0 ? (PARTS > 0 ? PARTS : -PARTS * (PKB ? num_mp : 1)) : 1;
  CK(cudaMemsetAsync(ctx->d_done, 0, sizeof(uint32_t) * num_n * counters, ctx->stream));
  CK(launch_persistent(kern, 2 * num_mp * a.rb_per_group, Cfg::THREADS, Cfg::SMEM_BYTES, ctx->stream, maps, a));
  ++ctx->launches;
  if (a.gtrace) {
    std::vector<unsigned long long> h(gtn);
    CK(cudaMemcpyAsync(h.data(), a.gtrace, gtn * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    char name[128];
    snprintf(name, sizeof name, "gpurun_out/res_gtrace_%d.txt", a.nsteps);
    FILE* f = fopen(name, "w");
    if (f) {
      const size_t grid = size_t(2 * (ctx->npad / 256) * a.rb_per_group);
      for (size_t i = 0; i < grid * 512; ++i)
        if (h[i]) fprintf(f, "%zu %zu %zu %llu\n", i / 512, (i / 8) % 64, i % 8, h[i]);
      fclose(f);
      snprintf(name, sizeof name, "gpurun_out/res_skew_%d.txt", a.nsteps);
      f = fopen(name, "w");
      if (f) {
        for (size_t i = 0; i < grid * 32; ++i)
          if (h[grid * 512 + i]) fprintf(f, "%zu %zu %llu\n", i / 32, i % 32, h[grid * 512 + i]);
        fclose(f);
      }
    }
  }
  if (a.trace) {
    std::vector<unsigned long long> h(size_t(16 * 4 * 4096));
    CK(cudaMemcpyAsync(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    FILE* f = fopen("gpurun_out/res_trace.txt", "w");
    if (f) {
      // parts 0, 1 of each step; the TS kernel also stamps parts 2, 3 (second region)
      const int nparts = (PARTS < 0 && SBG_TS_TRACE4) ? 4 : 2;
      for (int s = 0; s < a.nsteps; ++s)
        for (int c = 0; c < nparts; ++c) {
          const unsigned long long* r = &h[size_t(((c >> 1) * 2 * 4096 + s * 2 + (c & 1)) * 16)];
          fprintf(f, "%d %d", s, c);
          for (int k = 0; k < 16; ++k) fprintf(f, " %llu", r[k]);
          fprintf(f, "\n");
        }
      fclose(f);
    }
  }
  return SBG_OK;
}

void free_state(sbg_ctx* ctx) {
  ctx->ts_ok[0] = ctx->ts_ok[1] = false;  // freed buffers may be reallocated at the same addresses
  cudaFree(ctx->dX);
  cudaFree(ctx->dY);
  cudaFree(ctx->dP);
  cudaFree(ctx->dG[0]);
  cudaFree(ctx->dG[1]);
  cudaFree(ctx->dSign);
  cudaFree(ctx->dSignAll);
  ctx->dSignAll = nullptr;
  ctx->sign_all_bytes = 0;
  cudaFree(ctx->dE2);
  cudaFree(ctx->dE2p);
  ctx->dE2p = nullptr;
  cudaFree(ctx->dXs);
  cudaFree(ctx->dYs);
  cudaFree(ctx->dPs);
  cudaFree(ctx->dQ[0]);
  cudaFree(ctx->dQ[1]);
  ctx->dXs = ctx->dYs = ctx->dPs = nullptr;
  ctx->dQ[0] = ctx->dQ[1] = nullptr;
  cudaFree(ctx->dBest);
  cudaFree(ctx->d_done);
  ctx->d_done = nullptr;
  ctx->dX = ctx->dY = ctx->dP = nullptr;
  ctx->csr_sm_current = false;
  ctx->dG[0] = ctx->dG[1] = ctx->dSign = nullptr;
  ctx->dE2 = nullptr;
  ctx->dBest = nullptr;
  ctx->cap_rpad = 0;
}

// (Re)allocate the replica state for R replicas of the current instance.
int ensure_state(sbg_ctx* ctx, int64_t R) {
  if (ctx->kind == KIND_NONE) return ctx->fail(SBG_ERR_STATE, "couplings not set");
  ctx->csr_sm_current = false;  // every caller rewrites the replica-major state next
  if (R < 1) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "replica count must be >= 1");
  const int64_t rpad = round_up(R, PAD_R);
  if (rpad > (int64_t(1) << 30) / 4) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "too many replicas");
  if (rpad != ctx->cap_rpad) {
    free_state(ctx);
    const size_t st = sizeof(float) * size_t(rpad) * ctx->npad;
    const size_t pl = size_t(rpad) * ctx->npad;
    const size_t gpl = size_t(rpad) * gdim(ctx);  // B operand spans all spins (global when sharded)
    CK(cudaMalloc(&ctx->dX, st));
    CK(cudaMalloc(&ctx->dY, st));
    CK(cudaMalloc(&ctx->dP, st));
    CK(cudaMalloc(&ctx->dG[0], NPL * gpl));
    CK(cudaMalloc(&ctx->dG[1], NPL * gpl));
    CK(cudaMalloc(&ctx->dSign, pl));
    CK(cudaMalloc(&ctx->dE2, sizeof(unsigned long long) * rpad));
    CK(cudaMalloc(&ctx->dE2p, sizeof(unsigned long long) * rpad * FX_NA));
    CK(cudaMalloc(&ctx->dBest, 2 * sizeof(long long)));
    // per replica block / part / CTA pair (TS kernel: <= 5 parts x 8 pairs per 160 replicas)
    CK(cudaMalloc(&ctx->d_done, sizeof(uint32_t) * (rpad / 2 + 64)));
    CK(cudaMemsetAsync(ctx->dG[0], 0, NPL * gpl, ctx->stream));
    CK(cudaMemsetAsync(ctx->dG[1], 0, NPL * gpl, ctx->stream));
    CK(cudaMemsetAsync(ctx->dSign, 0, pl, ctx->stream));
    if (ctx->kind == KIND_CSR_I8) {
      // sized by rpad (not R): a later R in the same PAD_R bucket reuses these buffers, so the
      // leading dimension must cover every R that maps to this rpad
      ctx->rp = round_up(rpad, CSR_RCHUNK);
      const size_t sm = size_t(ctx->npad) * ctx->rp;
      for (float** a : {&ctx->dXs, &ctx->dYs, &ctx->dPs}) {
        CK(cudaMalloc(a, sizeof(float) * sm));
        CK(cudaMemsetAsync(*a, 0, sizeof(float) * sm, ctx->stream));
      }
      for (int b = 0; b < 2; ++b) {
        CK(cudaMalloc(&ctx->dQ[b], sizeof(int32_t) * sm));
        CK(cudaMemsetAsync(ctx->dQ[b], 0, sizeof(int32_t) * sm, ctx->stream));
      }
    }
    ctx->cap_rpad = rpad;
    if (ctx->kind == KIND_DENSE_I8 || ctx->kind == KIND_DENSE_FX) {
      for (int b = 0; b < 2; ++b) {
        int rc = encode_2d_u8(ctx, &ctx->tmG_sign[b], ctx->dG[b], gdim(ctx), rpad, 128, BN_SIGN);
        if (rc) return rc;
        rc = encode_2d_u8(ctx, &ctx->tmG_planes[b], ctx->dG[b], gdim(ctx), NPL * rpad, 128, BN_PLANE);
        if (rc) return rc;
      }
      int rc = encode_2d_u8(ctx, &ctx->tmSign, ctx->dSign, ctx->npad, rpad, 128, BN_SIGN);
      if (rc) return rc;
    }
  }
  ctx->R = R;
  ctx->rpad = rpad;
  ctx->g_mode = 0;
  if (ctx->kind == KIND_DENSE_I8 || ctx->kind == KIND_DENSE_FX) {
    constexpr int CW = TmaStepCfg<1, BN_SIGN, SIGN_STAGES, SIGN_NBUF>::CW;
    // Per B buffer b: output maps (the next step's B operand lands in the other buffer).
    CUtensorMap gout_sign[2], gout_planes[2];
    for (int b = 0; b < 2; ++b) {
      // stores of this shard's slab land at columns row0 + i; clip at the valid global width
      const uint64_t gvalid = uint64_t(ctx->sharded ? ctx->n_global : ctx->n);
      int rc = encode_2d(ctx, &gout_sign[b], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[b], gvalid, R, gdim(ctx), 128,
                         CW, CU_TENSOR_MAP_SWIZZLE_NONE);
      if (rc) return rc;
      rc = encode_2d(ctx, &gout_planes[b], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[b], gvalid, NPL * rpad,
                     gdim(ctx), 128, CW, CU_TENSOR_MAP_SWIZZLE_NONE);
      if (rc) return rc;
    }
    CUtensorMap X, Y, P;
    float* arrs[3] = {ctx->dX, ctx->dY, ctx->dP};
    CUtensorMap* outs[3] = {&X, &Y, &P};
    for (int a = 0; a < 3; ++a) {
      int rc = encode_2d(ctx, outs[a], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, arrs[a], ctx->n, R,
                         sizeof(float) * ctx->npad, 128, CW, CU_TENSOR_MAP_SWIZZLE_NONE);
      if (rc) return rc;
    }
    for (int cur = 0; cur < 2; ++cur) {
      for (int planes = 0; planes < 2; ++planes) {
        TmaMaps& mp = planes ? ctx->maps_planes[cur] : ctx->maps_sign[cur];
        mp.J = ctx->tmJ;
        // step parity 0 reads buffer cur and writes cur^1; parity 1 the reverse
        mp.Gin[0] = planes ? ctx->tmG_planes[cur] : ctx->tmG_sign[cur];
        mp.Gin[1] = planes ? ctx->tmG_planes[cur ^ 1] : ctx->tmG_sign[cur ^ 1];
        mp.Gout[0] = planes ? gout_planes[cur ^ 1] : gout_sign[cur ^ 1];
        mp.Gout[1] = planes ? gout_planes[cur] : gout_sign[cur];
        mp.X = X;
        mp.Y = Y;
        mp.P = P;
      }
      ctx->pmaps_planes[cur] = ctx->maps_planes[cur];
      ctx->maps_sign_cw8[cur] = ctx->maps_sign[cur];
      {
        const uint64_t gvalid = uint64_t(ctx->sharded ? ctx->n_global : ctx->n);
        TmaMaps& m8 = ctx->maps_sign_cw8[cur];
        int rc8 = encode_2d(ctx, &m8.Gout[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[cur ^ 1], gvalid, R, gdim(ctx),
                            128, 8, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (!rc8)
          rc8 = encode_2d(ctx, &m8.Gout[1], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[cur], gvalid, R, gdim(ctx), 128, 8,
                          CU_TENSOR_MAP_SWIZZLE_NONE);
        float* arrs8[3] = {ctx->dX, ctx->dY, ctx->dP};
        CUtensorMap* outs8[3] = {&m8.X, &m8.Y, &m8.P};
        for (int a8 = 0; a8 < 3 && !rc8; ++a8)
          rc8 = encode_2d(ctx, outs8[a8], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, arrs8[a8], ctx->n, R,
                          sizeof(float) * ctx->npad, 128, 8, CU_TENSOR_MAP_SWIZZLE_NONE);
        if (rc8) return rc8;
      }
      ctx->fxmaps_sign[cur] = ctx->maps_sign[cur];
      ctx->fxmaps_planes[cur] = ctx->maps_planes[cur];
      {
        TmaMaps& rm = ctx->rmaps_sign[cur];
        TmaMaps& rm160 = ctx->rmaps160_sign[cur];
        rm = ctx->maps_sign[cur];
        rm160 = ctx->maps_sign[cur];
        const uint64_t gvalid = uint64_t(ctx->sharded ? ctx->n_global : ctx->n);
        int rcr = SBG_OK;
        for (int par = 0; par < 2 && !rcr; ++par) {
          rcr = encode_2d_u8(ctx, &rm.Gin[par], ctx->dG[cur ^ par], ctx->npad, rpad, 128, 64);
          if (!rcr)
            rcr = encode_2d(ctx, &rm.Gout[par], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[cur ^ par ^ 1], gvalid, R,
                            gdim(ctx), 128, 128, CU_TENSOR_MAP_SWIZZLE_NONE);
          // B boxes of the last block may pass rpad: rows beyond are zero-filled (padding columns)
          if (!rcr) rcr = encode_2d_u8(ctx, &rm160.Gin[par], ctx->dG[cur ^ par], ctx->npad, rpad, 128, RES_NR / 2);
          if (!rcr)
            rcr = encode_2d(ctx, &rm160.Gout[par], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[cur ^ par ^ 1], gvalid, R,
                            gdim(ctx), 128, RES_NR, CU_TENSOR_MAP_SWIZZLE_NONE);
        }
        if (rcr) return rcr;
        if (ctx->dJ4) {  // e2m1 operands: G as [rpad][kpad / 2], two spins per byte
          const uint64_t gb = uint64_t(gdim(ctx) / 2), gv4 = (gvalid + 1) / 2;
          const int nrs[2] = {128, RES_NR};
          for (int w = 0; w < 2 && !rcr; ++w) {
            TmaMaps& qm = w ? ctx->qmaps160_sign[cur] : ctx->qmaps_sign[cur];
            qm = w ? rm160 : rm;
            qm.J = ctx->tmJ4;
            for (int par = 0; par < 2 && !rcr; ++par) {
              rcr = encode_2d_u8(ctx, &qm.Gin[par], ctx->dG[cur ^ par], gb, rpad, 128, nrs[w] / 2);
              if (!rcr)
                rcr = encode_2d(ctx, &qm.Gout[par], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[cur ^ par ^ 1], gv4, R,
                                gb, 64, nrs[w], CU_TENSOR_MAP_SWIZZLE_NONE);
            }
          }
          for (int wv = 0; wv < 2 && !rcr; ++wv) {
            TmaMaps& pq = wv ? ctx->pq128maps_sign[cur] : ctx->pqmaps_sign[cur];
            pq = ctx->maps_sign[cur];
            pq.J = ctx->tmJ4;
            for (int par = 0; par < 2 && !rcr; ++par) {
              rcr = encode_2d_u8(ctx, &pq.Gin[par], ctx->dG[cur ^ par], gb, rpad, 128, (wv ? 128 : NPAIR_SIGN) / 2);
              if (!rcr)
                rcr = encode_2d(ctx, &pq.Gout[par], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[cur ^ par ^ 1], gv4, R,
                                gb, 64, 16, CU_TENSOR_MAP_SWIZZLE_NONE);
            }
          }
          if (rcr) return rcr;
        }
      }
      for (int par = 0; par < 2; ++par) {
        int rc = encode_2d_u8(ctx, &ctx->pmaps_planes[cur].Gin[par], ctx->dG[cur ^ par], ctx->npad, NPL * rpad, 128,
                              NPAIR_PLANE / 2);
        if (rc) return rc;
        rc = encode_2d_u8(ctx, &ctx->fxmaps_sign[cur].Gin[par], ctx->dG[cur ^ par], ctx->npad, rpad, 128, BN_FX_SIGN);
        if (rc) return rc;
        rc = encode_2d_u8(ctx, &ctx->fxmaps_planes[cur].Gin[par], ctx->dG[cur ^ par], ctx->npad, NPL * rpad, 128,
                          BN_FX_PLANE);
        if (rc) return rc;
        ctx->fxq_planes64[cur] = ctx->maps_planes[cur];
        ctx->fxq_planes32[cur] = ctx->fxmaps_planes[cur];
      }
      for (int par = 0; par < 2; ++par) {
        int rc = encode_2d_u8(ctx, &ctx->fxq_planes64[cur].Gin[par], ctx->dG[cur ^ par], ctx->npad, NPL * rpad, 64,
                              BN_FX_PLANE_W, CU_TENSOR_MAP_SWIZZLE_64B);
        if (rc) return rc;
        rc = encode_2d_u8(ctx, &ctx->fxq_planes32[cur].Gin[par], ctx->dG[cur ^ par], ctx->npad, NPL * rpad, 64,
                          BN_FX_PLANE, CU_TENSOR_MAP_SWIZZLE_64B);
        if (rc) return rc;
      }
    }
  }
  const size_t st = sizeof(float) * size_t(rpad) * ctx->npad;
  CK(cudaMemsetAsync(ctx->dX, 0, st, ctx->stream));
  CK(cudaMemsetAsync(ctx->dY, 0, st, ctx->stream));
  CK(cudaMemsetAsync(ctx->dP, 0, st, ctx->stream));
  return SBG_OK;
}

int prep_planes(sbg_ctx* ctx, const float* x, uint8_t* G, int nplanes, int64_t R, int64_t rpad,
                bool into_global = false) {
  const size_t total = size_t(rpad) * ctx->npad;
  const int64_t g_ld = into_global ? gdim(ctx) : ctx->npad;
  const int64_t col0 = into_global && ctx->sharded ? ctx->row0 : 0;
  prep_planes_kernel<<<grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(
      x, G, int32_t(ctx->n), int32_t(ctx->npad), ctx->npad, int32_t(R), int32_t(rpad), nplanes, g_ld, col0);
  CK(cudaGetLastError());
  ++ctx->launches;
  return SBG_OK;
}

StepArgs base_args(const sbg_ctx* ctx, int BN, int64_t R, int64_t rpad) {
  StepArgs a;
  std::memset(&a, 0, sizeof a);
  a.n = int32_t(ctx->n);
  a.npad = int32_t(ctx->npad);
  a.R = int32_t(R);
  a.rpad = int32_t(rpad);
  a.num_m = int32_t(ctx->npad / 128);
  a.num_n = int32_t(rpad / BN);
  a.kpad = int32_t(ctx->sharded ? ctx->kpad : ctx->npad);
  a.ld = ctx->npad;
  return a;
}

int validate_params(sbg_ctx* ctx, const sbg_params* p) {
  // validate() engine.cpp:16-21 (dt/c are resolved here, so both must be > 0)
  if (!p) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "params is null");
  if (p->variant < SBG_BSB || p->variant > SBG_GDSB) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "unknown variant");
  if (p->steps < 1) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "step count M must be >= 1");
  if (!(p->dt > 0.0)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "dt must be positive");
  if (!(p->c > 0.0)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "c must be positive");
  if (!(p->a >= 0.0)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "A must be >= 0");
  if (p->steps >= (uint64_t(1) << 24))
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "M must be < 2^24 (fp32 step denominator)");
  return SBG_OK;
}


// ------------------------------------------------------------- device generators

enum { GEN_HASH = 0, GEN_EXACT = 1 };

// xoshiro jump matrices T^(2^k) (gen_dense.cuh), computed once per process.
const std::vector<uint64_t>& jump_matrices() {
  static const std::vector<uint64_t> m = gen_jump_matrices(GEN_MAXK);
  return m;
}

// The e2m1 copy of a dense int8 J (rows x kpad), kept only if every entry is e2m1-exact.
int build_q4(sbg_ctx* ctx, int64_t rows, int64_t kpad) {
  cudaFree(ctx->dJ4);
  ctx->dJ4 = nullptr;
  if (getenv_is0("SBG_Q4")) return SBG_OK;
  const size_t bytes = size_t(rows) * size_t(kpad / 2);
  unsigned* bad = nullptr;
  CK(cudaMalloc(&ctx->dJ4, bytes));
  CK(cudaMalloc(&bad, sizeof(unsigned)));
  CK(cudaMemsetAsync(bad, 0, sizeof(unsigned), ctx->stream));
  pack_e2m1_kernel<<<grid_for(ctx, bytes / 16, 256), 256, 0, ctx->stream>>>(ctx->dJ, ctx->dJ4, bytes, bad);
  ++ctx->launches;
  unsigned h = 1;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bad, sizeof h, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(bad);
  if (e != cudaSuccess) return ctx->fail(SBG_ERR_CUDA, "e2m1 packing: %s", cudaGetErrorString(e));
  if (h) {
    cudaFree(ctx->dJ4);
    ctx->dJ4 = nullptr;
    return SBG_OK;
  }
  return encode_2d_u8(ctx, &ctx->tmJ4, ctx->dJ4, uint64_t(kpad / 2), uint64_t(rows), 128, 128);
}

// Allocates this context's dense int8 rows (all rows when world == 1, else the
// row-shard layout of sbg_set_couplings_rows_i8) and fills them on the device:
// GEN_EXACT = gen_random_dense's draw order (gen_dense.cuh), GEN_HASH = the
// counter-based i.i.d. +-1 instance.
int gen_rows_common(sbg_ctx* ctx, int64_t n_global, int32_t world, int32_t rank, uint64_t seed, int which) {
  if (n_global < 2 || world < 1 || world > 8 || rank < 0 || rank >= world)
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad arguments");
  const int64_t total = n_global * (n_global - 1) / 2;
  if (which == GEN_EXACT && (total >> GEN_MAXK) != 0) return ctx->fail(SBG_ERR_UNSUPPORTED, "n too large");
  CK(cudaSetDevice(ctx->device));
  cudaStreamSynchronize(ctx->stream);
  free_state(ctx);
  cudaFree(ctx->dJ);
  cudaFree(ctx->dJ4);
  ctx->dJ4 = nullptr;
  ctx->dJ = nullptr;
  const bool shard = world > 1;
  const int64_t kpad = shard ? round_up(n_global, int64_t(256) * world) : round_up(n_global, PAD_N);
  const int64_t rows = shard ? kpad / world : kpad;
  const int64_t row0 = shard ? int64_t(rank) * rows : 0;
  const int64_t valid = std::max<int64_t>(0, std::min<int64_t>(rows, n_global - row0));
  if (valid == 0) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "rank owns no spins");
  CK(cudaMalloc(&ctx->dJ, size_t(rows) * kpad));
  if (which == GEN_HASH) {
    const uint64_t work = uint64_t(rows) * kpad / 16;
    gen_hash_pm1_kernel<<<int(std::min<uint64_t>((work + 255) / 256, uint64_t(ctx->sms) * 32)), 256, 0,
                          ctx->stream>>>(ctx->dJ, n_global, row0, rows, kpad, seed);
    CK(cudaGetLastError());
    ++ctx->launches;
  } else {
    int seg = GEN_SEG;
    if (const char* e = getenv("SBG_GEN_SEG")) seg = std::max(8, atoi(e) / 8 * 8);  // dev knob (tests)
    int kmax = 1;
    while (kmax < GEN_MAXK && (uint64_t(total) >> kmax) != 0) ++kmax;
    const auto& mats = jump_matrices();
    ulonglong4* dmat = nullptr;
    CK(cudaMalloc(&dmat, sizeof(uint64_t) * 1024 * kmax));
    CK(cudaMemcpyAsync(dmat, mats.data(), sizeof(uint64_t) * 1024 * kmax, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->dJ, 0, size_t(rows) * kpad, ctx->stream));
    const int64_t r1 = row0 + valid;
    const int64_t up_threads = valid * ((n_global + seg - 1) / seg);
    gen_dense_upper_kernel<<<unsigned((up_threads + 127) / 128), 128, 0, ctx->stream>>>(
        ctx->dJ, kpad, n_global, row0, r1, dmat, kmax, seed, seg);
    CK(cudaGetLastError());
    ++ctx->launches;
    if (!shard) {
      mirror_lower_kernel<<<dim3(unsigned(kpad / 64), unsigned(kpad / 64)), 256, 0, ctx->stream>>>(ctx->dJ, kpad,
                                                                                                  n_global);
    } else {
      const int64_t st_threads = r1 * ((valid + seg - 1) / seg);
      gen_dense_strip_kernel<<<unsigned((st_threads + 127) / 128), 128, 0, ctx->stream>>>(
          ctx->dJ, kpad, n_global, row0, r1, dmat, kmax, seed, seg);
    }
    CK(cudaGetLastError());
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(dmat);
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->kind = KIND_DENSE_I8;
  ctx->energy_scale = 1.0;
  ctx->sharded = shard;
  ctx->n = shard ? valid : n_global;
  ctx->npad = rows;
  ctx->n_global = n_global;
  ctx->kpad = kpad;
  ctx->row0 = row0;
  ctx->num_m_total = kpad / 128;
  ctx->done_base = 0;
  ctx->peer_g0.clear();
  ctx->peer_g1.clear();
  ctx->peer_done.clear();
  const int rc = encode_2d_u8(ctx, &ctx->tmJ, ctx->dJ, kpad, rows, 128, 128);
  return rc ? rc : build_q4(ctx, rows, kpad);
}


// ------------------------------------------------------------------ spectral (auto_tune)

int make_jview(sbg_ctx* ctx, JView* v) {
  if (ctx->kind == KIND_NONE) return ctx->fail(SBG_ERR_STATE, "couplings not set");
  if (ctx->sharded) return ctx->fail(SBG_ERR_UNSUPPORTED, "spectral estimation of a row shard");
  *v = JView{};
  v->n = ctx->n;
  if (ctx->kind == KIND_CSR_I8) {
    v->kind = JV_CSR_I8;
    v->rowptr = ctx->d_rowptr;
    v->col = ctx->d_col;
    v->val = ctx->d_val;
  } else {
    v->kind = ctx->kind == KIND_DENSE_I8 ? JV_DENSE_I8 : JV_DENSE_FX;
    v->J = ctx->dJ;
    v->ld = ctx->npad;
    v->plane = ctx->npad * ctx->npad;
    v->scale = std::ldexp(1.0, -ctx->fx_shift);
  }
  return SBG_OK;
}

// Row sums of J^2 (off-diagonal) and |J| on the device; sum_sq summed on the host in
// row order, beta = max row sum (exact for integer J in any order).
int row_stats(sbg_ctx* ctx, const JView& jv, double* sum_sq, double* beta) {
  double* d = nullptr;
  CK(cudaMalloc(&d, sizeof(double) * 2 * jv.n));
  row_stats_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(jv, d, d + jv.n);
  ++ctx->launches;
  std::vector<double> h(size_t(2 * jv.n));
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, sizeof(double) * 2 * jv.n, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d);
  if (e != cudaSuccess) return ctx->fail(SBG_ERR_CUDA, "row statistics: %s", cudaGetErrorString(e));
  double sq = 0.0, b = 0.0;
  for (int64_t i = 0; i < jv.n; ++i) {
    sq += h[size_t(i)];
    b = std::max(b, h[size_t(jv.n + i)]);
  }
  *sum_sq = sq;
  *beta = b;
  return SBG_OK;
}

struct PowerOutcome {
  double lambda = 0.0, residual = 0.0;
  uint64_t iterations = 0;
  bool converged = false;
};

// One end of the spectrum (spectral.cpp:50-118) as one cooperative launch.
int power_end(sbg_ctx* ctx, const JView& jv, double beta, double sign, double tol, uint64_t max_iters,
              PowerOutcome* out, double* v_out) {
  const int64_t n = jv.n;
  double* buf = nullptr;
  const size_t nb = size_t(3 * n + 8);
  CK(cudaMalloc(&buf, sizeof(double) * nb + 64));
  CK(cudaMemsetAsync(buf, 0, sizeof(double) * nb + 64, ctx->stream));
  PowerArgs a{};
  a.J = jv;
  a.beta = beta;
  a.sign = sign;
  a.tol = tol;
  a.v_init = 1.0 / std::sqrt(static_cast<double>(n));
  a.max_iters = max_iters;
  a.v[0] = buf;
  a.v[1] = buf + n;
  a.jv = buf + 2 * n;
  a.result = buf + 3 * n;             // 5 doubles
  a.bar = reinterpret_cast<unsigned long long*>(buf + 3 * n + 6);
  a.ctrl = reinterpret_cast<int*>(buf + 3 * n + 7);
  CK(cudaFuncSetAttribute(power_iteration_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PI_SMEM_BYTES));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, power_iteration_kernel, PI_THREADS, PI_SMEM_BYTES));
  if (per_sm < 1) {
    cudaFree(buf);
    return ctx->fail(SBG_ERR_CUDA, "power iteration kernel cannot be resident");
  }
  void* params[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(power_iteration_kernel), dim3(ctx->sms),
                                              dim3(PI_THREADS), params, PI_SMEM_BYTES, ctx->stream);
  ++ctx->launches;
  double res[5] = {0, 0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(res, a.result, sizeof res, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess && v_out)
    e = cudaMemcpy(v_out, a.v[int(res[4])], sizeof(double) * n, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (e != cudaSuccess) return ctx->fail(SBG_ERR_CUDA, "power iteration: %s", cudaGetErrorString(e));
  out->lambda = res[0];
  out->residual = res[1];
  out->iterations = uint64_t(res[2]);
  out->converged = res[3] != 0.0;
  return SBG_OK;
}

}  // namespace

extern "C" {

int sbg_abi_version(void) { return SBG_ABI_VERSION; }

const char* sbg_strerror(int code) {
  switch (code) {
    case SBG_OK: return "ok";
    case SBG_ERR_INVALID_ARGUMENT: return "invalid argument";
    case SBG_ERR_OUT_OF_MEMORY: return "out of device memory";
    case SBG_ERR_CUDA: return "CUDA error";
    case SBG_ERR_NCCL: return "NCCL error";
    case SBG_ERR_STATE: return "invalid call order";
    case SBG_ERR_UNSUPPORTED: return "unsupported";
    case SBG_ERR_CONVERGENCE: return "eigenvalue estimation did not converge";
  }
  return "unknown";
}

int sbg_create(int device, sbg_ctx** out) {
  if (!out) return SBG_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return SBG_ERR_CUDA;
  if (device < 0 || device >= count) return SBG_ERR_INVALID_ARGUMENT;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SBG_ERR_CUDA;
  if (prop.major != 10) return SBG_ERR_UNSUPPORTED;  // sm_100a only
  if (cudaSetDevice(device) != cudaSuccess) return SBG_ERR_CUDA;
  auto* ctx = new sbg_ctx();
  ctx->device = device;
  ctx->sms = prop.multiProcessorCount;
  ctx->device_name = prop.name;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return SBG_ERR_CUDA;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  for (auto& e : ctx->evc) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking) != cudaSuccess) {
    sbg_destroy(ctx);
    return SBG_ERR_CUDA;
  }
  *out = ctx;
  return SBG_OK;
}

void sbg_destroy(sbg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  free_state(ctx);
  cudaFree(ctx->d_arep);
  cudaFree(ctx->d_ready);
  cudaFree(ctx->d_fpart);
  cudaFree(ctx->d_kdone);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_fused);
  cudaFree(ctx->dJ);
  cudaFree(ctx->dJ4);
  ctx->dJ4 = nullptr;
  cudaFree(ctx->d_rowptr);
  cudaFree(ctx->d_col);
  cudaFree(ctx->d_val);
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  for (auto& e : ctx->evc) cudaEventDestroy(e);
  if (ctx->cstream) {
    cudaStreamSynchronize(ctx->cstream);
    cudaStreamDestroy(ctx->cstream);
  }
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* sbg_last_error(const sbg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
int sbg_device_sm_count(const sbg_ctx* ctx) { return ctx ? ctx->sms : 0; }
const char* sbg_device_name(const sbg_ctx* ctx) { return ctx ? ctx->device_name.c_str() : ""; }
int64_t sbg_n(const sbg_ctx* ctx) { return ctx ? ctx->n : 0; }
int sbg_couplings_e2m1(const sbg_ctx* ctx) { return ctx && ctx->dJ4 ? 1 : 0; }
int64_t sbg_kernel_launches(const sbg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int sbg_set_couplings_dense_i8(sbg_ctx* ctx, int64_t n, const int8_t* J) {
  CHECK_CTX(ctx);
  if (n < 1 || !J) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "instance size must be >= 1");
  // IsingInstance invariants (model.cpp:54-68)
  for (int64_t i = 0; i < n; ++i) {
    if (J[i * n + i] != 0) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling diagonal must be zero");
    for (int64_t j = i + 1; j < n; ++j)
      if (J[i * n + j] != J[j * n + i])
        return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling matrix must be symmetric");
    for (int64_t j = 0; j < n; ++j)
      if (J[i * n + j] == -128)
        return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "int8 couplings must lie in [-127, 127]");
  }
  CK(cudaSetDevice(ctx->device));
  cudaStreamSynchronize(ctx->stream);
  free_state(ctx);
  cudaFree(ctx->dJ);
  cudaFree(ctx->dJ4);
  ctx->dJ4 = nullptr;
  ctx->dJ = nullptr;
  const int64_t npad = round_up(n, PAD_N);
  CK(cudaMalloc(&ctx->dJ, size_t(npad) * npad));
  CK(cudaMemsetAsync(ctx->dJ, 0, size_t(npad) * npad, ctx->stream));
  CK(cudaMemcpy2DAsync(ctx->dJ, npad, J, n, n, n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->n = n;
  ctx->npad = npad;
  ctx->kind = KIND_DENSE_I8;
  ctx->energy_scale = 1.0;
  const int rc = encode_2d_u8(ctx, &ctx->tmJ, ctx->dJ, npad, npad, 128, 128);
  return rc ? rc : build_q4(ctx, npad, npad);
}

int sbg_set_couplings_dense_f64(sbg_ctx* ctx, int64_t n, const double* J) {
  CHECK_CTX(ctx);
  if (n < 1 || !J) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "instance size must be >= 1");
  std::vector<int8_t> q(size_t(n) * n);
  bool integral = true;
  for (int64_t k = 0; k < n * n && integral; ++k) {
    const double v = J[k];
    integral = (v == std::floor(v)) && v >= -127.0 && v <= 127.0;
    q[size_t(k)] = integral ? static_cast<int8_t>(v) : 0;
  }
  if (integral) return sbg_set_couplings_dense_i8(ctx, n, q.data());
  // real-valued couplings: the fixed-point path (rounded to fp32 first, as the state is fp32)
  std::vector<float> f(size_t(n) * n);
  for (int64_t k = 0; k < n * n; ++k) f[size_t(k)] = static_cast<float>(J[k]);
  return sbg_set_couplings_dense_f32(ctx, n, f.data());
}

int sbg_set_couplings_dense_f32(sbg_ctx* ctx, int64_t n, const float* J) {
  CHECK_CTX(ctx);
  if (n < 1 || !J) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "instance size must be >= 1");
  // IsingInstance invariants (model.cpp:54-68)
  float amax = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    if (J[i * n + i] != 0.0f) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling diagonal must be zero");
    for (int64_t j = i + 1; j < n; ++j)
      if (J[i * n + j] != J[j * n + i]) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling matrix must be symmetric");
    for (int64_t j = 0; j < n; ++j) {
      if (!std::isfinite(J[i * n + j])) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "couplings must be finite");
      amax = std::max(amax, std::fabs(J[i * n + j]));
    }
  }
  if (amax == 0.0f) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "degenerate instance: all couplings zero");
  // J_int = rint(J * 2^s) with |J_int| <= 2^23 - 1 (24-bit two's complement in 3 byte planes),
  // and the per-weight s32 accumulators must not overflow: 3 * 255 * 255 * n < 2^31.
  if (3.0 * 255.0 * 255.0 * double(n) >= 2147483648.0)
    return ctx->fail(SBG_ERR_UNSUPPORTED, "real-valued couplings supported up to n = 11000");
  int shift = 0;
  while (std::ldexp(double(amax), shift + 1) <= 8388607.0 && shift < 60) ++shift;
  while (std::ldexp(double(amax), shift) > 8388607.0) --shift;
  const int64_t npad = round_up(n, PAD_N);
  std::vector<uint8_t> planes(size_t(FX_NA) * npad * npad, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const int32_t qv = static_cast<int32_t>(std::nearbyint(std::ldexp(double(J[i * n + j]), shift)));
      for (int a = 0; a < FX_NA; ++a)
        planes[size_t(a) * npad * npad + size_t(i) * npad + j] = static_cast<uint8_t>(uint32_t(qv) >> (8 * a));
    }
  CK(cudaSetDevice(ctx->device));
  cudaStreamSynchronize(ctx->stream);
  free_state(ctx);
  cudaFree(ctx->dJ);
  cudaFree(ctx->dJ4);
  ctx->dJ4 = nullptr;
  ctx->dJ = nullptr;
  CK(cudaMalloc(&ctx->dJ, planes.size()));
  CK(cudaMemcpy(ctx->dJ, planes.data(), planes.size(), cudaMemcpyHostToDevice));
  ctx->n = n;
  ctx->npad = npad;
  ctx->kind = KIND_DENSE_FX;
  ctx->fx_shift = shift;
  ctx->energy_scale = std::ldexp(1.0, -shift);
  int rc = encode_2d_u8(ctx, &ctx->tmJ, ctx->dJ, npad, FX_NA * npad, 128, 128);
  if (rc == SBG_OK) rc = encode_2d_u8(ctx, &ctx->tmJfx64, ctx->dJ, npad, FX_NA * npad, 64, 128, CU_TENSOR_MAP_SWIZZLE_64B);
  for (int a = 0; a < FX_NA && rc == SBG_OK; ++a)
    rc = encode_2d_u8(ctx, &ctx->tmJplane[a], ctx->dJ + size_t(a) * npad * npad, npad, npad, 128, 128);
  return rc;
}

int sbg_coupling_scale_exp(const sbg_ctx* ctx) { return ctx && ctx->kind == KIND_DENSE_FX ? ctx->fx_shift : 0; }

int sbg_gen_couplings_dense_pm1(sbg_ctx* ctx, int64_t n, uint64_t seed) {
  CHECK_CTX(ctx);
  if (n < 2) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "random dense instance needs n >= 2");
  return gen_rows_common(ctx, n, 1, 0, seed, GEN_EXACT);
}

int sbg_set_couplings_csr_i8(sbg_ctx* ctx, int64_t n, int64_t nnz, const int32_t* rowptr,
                             const int32_t* col, const int8_t* val) {
  CHECK_CTX(ctx);
  if (n < 1 || nnz < 0 || !rowptr || (nnz > 0 && (!col || !val)))
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad CSR arguments");
  if (rowptr[0] != 0 || rowptr[n] != nnz) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad CSR row pointer");
  for (int64_t i = 0; i < n; ++i) {
    if (rowptr[i + 1] < rowptr[i]) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "CSR row pointer not monotone");
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      if (col[k] < 0 || col[k] >= n) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling index out of range");
      if (col[k] == i) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling diagonal must be zero");
      if (k > rowptr[i] && col[k] <= col[k - 1])
        return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "CSR columns must be strictly ascending");
      if (val[k] == -128) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "int8 couplings must lie in [-127, 127]");
    }
  }
  CK(cudaSetDevice(ctx->device));
  cudaStreamSynchronize(ctx->stream);
  free_state(ctx);
  cudaFree(ctx->dJ);
  cudaFree(ctx->dJ4);
  ctx->dJ4 = nullptr;
  cudaFree(ctx->d_rowptr);
  cudaFree(ctx->d_col);
  cudaFree(ctx->d_val);
  ctx->dJ = nullptr;
  ctx->d_rowptr = ctx->d_col = nullptr;
  ctx->d_val = nullptr;
  CK(cudaMalloc(&ctx->d_rowptr, sizeof(int32_t) * (n + 1)));
  CK(cudaMalloc(&ctx->d_col, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  CK(cudaMalloc(&ctx->d_val, std::max<int64_t>(nnz, 1)));
  CK(cudaMemcpy(ctx->d_rowptr, rowptr, sizeof(int32_t) * (n + 1), cudaMemcpyHostToDevice));
  if (nnz) {
    CK(cudaMemcpy(ctx->d_col, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_val, val, nnz, cudaMemcpyHostToDevice));
  }
  ctx->n = n;
  ctx->npad = round_up(n, 32);
  ctx->nnz = nnz;
  ctx->kind = KIND_CSR_I8;
  ctx->energy_scale = 1.0;
  return SBG_OK;
}

namespace {
// Both-triangle CSR with ascending columns from an upper-or-lower edge list (val = J_ij).
int csr_from_pairs(sbg_ctx* ctx, int64_t n, const std::vector<int64_t>& a, const std::vector<int64_t>& b,
                   const std::vector<int8_t>& v) {
  std::vector<int32_t> rowptr(size_t(n) + 1, 0);
  for (size_t k = 0; k < a.size(); ++k) {
    ++rowptr[size_t(a[k]) + 1];
    ++rowptr[size_t(b[k]) + 1];
  }
  for (int64_t r = 0; r < n; ++r) rowptr[size_t(r) + 1] += rowptr[size_t(r)];
  const int64_t nnz = rowptr[size_t(n)];
  std::vector<int32_t> fill(rowptr.begin(), rowptr.end() - 1), col(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  std::vector<int8_t> val(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  for (size_t k = 0; k < a.size(); ++k) {
    int32_t& fa = fill[size_t(a[k])];
    col[size_t(fa)] = int32_t(b[k]);
    val[size_t(fa++)] = v[k];
    int32_t& fb = fill[size_t(b[k])];
    col[size_t(fb)] = int32_t(a[k]);
    val[size_t(fb++)] = v[k];
  }
  std::vector<std::pair<int32_t, int8_t>> row;
  for (int64_t r = 0; r < n; ++r) {
    const int32_t lo = rowptr[size_t(r)], hi = rowptr[size_t(r) + 1];
    row.clear();
    for (int32_t k = lo; k < hi; ++k) row.emplace_back(col[size_t(k)], val[size_t(k)]);
    std::sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    for (int32_t k = lo; k < hi; ++k) {
      col[size_t(k)] = row[size_t(k - lo)].first;
      val[size_t(k)] = row[size_t(k - lo)].second;
    }
  }
  return sbg_set_couplings_csr_i8(ctx, n, nnz, rowptr.data(), col.data(), val.data());
}

uint64_t pair_key(int64_t i, int64_t j) {  // model.cpp pair_key: unordered pair
  const uint64_t a = uint64_t(std::min(i, j)), b = uint64_t(std::max(i, j));
  return (a << 32) ^ b;
}
}  // namespace

int sbg_set_couplings_graph(sbg_ctx* ctx, int64_t n, int64_t m, const int64_t* ei, const int64_t* ej,
                            const int64_t* w, int64_t* total_weight) {
  CHECK_CTX(ctx);
  if (n < 1) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "instance size must be >= 1");
  if (m < 0 || (m > 0 && (!ei || !ej || !w))) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad edge arrays");
  if (n > INT32_MAX) return ctx->fail(SBG_ERR_UNSUPPORTED, "n beyond int32 CSR indices");
  // CutGraph invariants (model.cpp:91-103), in input order
  std::unordered_set<uint64_t> seen;
  seen.reserve(size_t(m));
  std::vector<int64_t> a(static_cast<size_t>(m)), b(static_cast<size_t>(m));
  std::vector<int8_t> v(static_cast<size_t>(m));
  long long W = 0;
  for (int64_t k = 0; k < m; ++k) {
    if (ei[k] < 0 || ej[k] < 0 || ei[k] >= n || ej[k] >= n)
      return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "edge endpoint out of range");
    if (ei[k] == ej[k]) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "self-loops are not allowed");
    if (!seen.insert(pair_key(ei[k], ej[k])).second)
      return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "duplicate edge (%lld, %lld)", (long long)ei[k], (long long)ej[k]);
    if (w[k] < -127 || w[k] > 127)
      return ctx->fail(SBG_ERR_UNSUPPORTED, "edge weight %lld outside the int8 coupling range", (long long)w[k]);
    a[size_t(k)] = ei[k];
    b[size_t(k)] = ej[k];
    v[size_t(k)] = int8_t(-w[k]);  // maxcut_to_ising (model.cpp:134-142): J = -w
    W += w[k];
  }
  const int rc = csr_from_pairs(ctx, n, a, b, v);
  if (rc == SBG_OK && total_weight) *total_weight = W;
  return rc;
}

int sbg_set_couplings_entries_f64(sbg_ctx* ctx, int64_t n, int64_t m, const int64_t* ei, const int64_t* ej,
                                  const double* value) {
  CHECK_CTX(ctx);
  if (n < 1) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "instance size must be >= 1");
  if (m < 0 || (m > 0 && (!ei || !ej || !value))) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad entry arrays");
  // IsingInstance::from_entries (model.cpp:70-86), in input order
  std::unordered_set<uint64_t> seen;
  seen.reserve(size_t(m));
  bool integral = true;
  for (int64_t k = 0; k < m; ++k) {
    if (ei[k] < 0 || ej[k] < 0 || ei[k] >= n || ej[k] >= n)
      return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling index out of range");
    if (ei[k] == ej[k]) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "diagonal couplings are not allowed");
    if (!seen.insert(pair_key(ei[k], ej[k])).second)
      return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "duplicate coupling entry (%lld, %lld)", (long long)ei[k],
                       (long long)ej[k]);
    const double x = value[k];
    integral = integral && x == std::floor(x) && x >= -127.0 && x <= 127.0;
  }
  if (integral && n <= INT32_MAX && double(2 * m) < double(n) * double(n) / 16.0) {
    std::vector<int64_t> a, b;
    std::vector<int8_t> v;
    for (int64_t k = 0; k < m; ++k)
      if (value[k] != 0.0) {
        a.push_back(ei[k]);
        b.push_back(ej[k]);
        v.push_back(int8_t(value[k]));
      }
    return csr_from_pairs(ctx, n, a, b, v);
  }
  if (double(n) * double(n) > 4e10) return ctx->fail(SBG_ERR_UNSUPPORTED, "dense real-valued instance too large");
  std::vector<double> J(size_t(n) * size_t(n), 0.0);
  for (int64_t k = 0; k < m; ++k) {
    J[size_t(ei[k]) * size_t(n) + size_t(ej[k])] = value[k];
    J[size_t(ej[k]) * size_t(n) + size_t(ei[k])] = value[k];
  }
  return sbg_set_couplings_dense_f64(ctx, n, J.data());
}

// CSR: sbg_advance leaves the state in the spin-major working copies (the next advance
// continues from them with no transposes); anything that reads the replica-major x, y, p
// first brings them up to date (three transposes, once).
static int csr_sync(sbg_ctx* ctx) {
  if (ctx->kind != KIND_CSR_I8 || !ctx->csr_sm_current) return SBG_OK;
  const dim3 tb(32, 8);
  const dim3 tg_out(unsigned((ctx->R + 31) / 32), unsigned((ctx->n + 31) / 32));
  float* rm[3] = {ctx->dX, ctx->dY, ctx->dP};
  float* sm[3] = {ctx->dXs, ctx->dYs, ctx->dPs};
  for (int a = 0; a < 3; ++a) {
    transpose_f32_kernel<<<tg_out, tb, 0, ctx->stream>>>(sm[a], rm[a], int32_t(ctx->n), int32_t(ctx->R), ctx->rp,
                                                         ctx->npad);
    CK(cudaGetLastError());
    ++ctx->launches;
  }
  ctx->csr_sm_current = false;
  return SBG_OK;
}

int sbg_set_state(sbg_ctx* ctx, int64_t R, const float* x, const float* y, const float* p) {
  CHECK_CTX(ctx);
  if (!x || !y) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "x and y are required");
  CK(cudaSetDevice(ctx->device));
  int rc = ensure_state(ctx, R);
  if (rc) return rc;
  const size_t pitch = sizeof(float) * ctx->npad, w = sizeof(float) * ctx->n;
  CK(cudaMemcpy2DAsync(ctx->dX, pitch, x, w, w, R, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpy2DAsync(ctx->dY, pitch, y, w, w, R, cudaMemcpyHostToDevice, ctx->stream));
  if (p) {
    CK(cudaMemcpy2DAsync(ctx->dP, pitch, p, w, w, R, cudaMemcpyHostToDevice, ctx->stream));
  } else {
    const size_t cnt = size_t(ctx->rpad) * ctx->npad;
    fill_f32_kernel<<<grid_for(ctx, cnt, 256), 256, 0, ctx->stream>>>(ctx->dP, cnt, 1.0f);
    CK(cudaGetLastError());
    ++ctx->launches;
  }
  return SBG_OK;
}

int sbg_init_state(sbg_ctx* ctx, int64_t R, int32_t mode, uint64_t master, uint64_t tag, int64_t offset) {
  CHECK_CTX(ctx);
  if (mode < 0 || mode > 2) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "unknown init mode");
  CK(cudaSetDevice(ctx->device));
  int rc = ensure_state(ctx, R);
  if (rc) return rc;
  const int blocks = int((R + INIT_THREADS - 1) / INIT_THREADS);
  init_state_kernel<<<blocks, INIT_THREADS, 0, ctx->stream>>>(
      ctx->dX, ctx->dY, ctx->dP, int32_t(ctx->n), ctx->npad, int32_t(R), mode, master, tag, offset,
      ctx->sharded ? ctx->n_global : ctx->n, ctx->sharded ? ctx->row0 : 0);
  CK(cudaGetLastError());
  ++ctx->launches;
  return SBG_OK;
}

int sbg_init_state_seeds(sbg_ctx* ctx, int64_t R, int32_t mode, const uint64_t* seeds) {
  CHECK_CTX(ctx);
  if (mode < 0 || mode > 2 || !seeds) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad init arguments");
  CK(cudaSetDevice(ctx->device));
  int rc = ensure_state(ctx, R);
  if (rc) return rc;
  uint64_t* dseeds = nullptr;
  CK(cudaMalloc(&dseeds, sizeof(uint64_t) * size_t(R)));
  CK(cudaMemcpyAsync(dseeds, seeds, sizeof(uint64_t) * size_t(R), cudaMemcpyHostToDevice, ctx->stream));
  const int blocks = int((R + INIT_THREADS - 1) / INIT_THREADS);
  init_state_kernel<<<blocks, INIT_THREADS, 0, ctx->stream>>>(
      ctx->dX, ctx->dY, ctx->dP, int32_t(ctx->n), ctx->npad, int32_t(R), mode, 0, 0, 0,
      ctx->sharded ? ctx->n_global : ctx->n, ctx->sharded ? ctx->row0 : 0, dseeds);
  CK(cudaGetLastError());
  ++ctx->launches;
  CK(cudaStreamSynchronize(ctx->stream));
  cudaFree(dseeds);
  return SBG_OK;
}

int sbg_get_state(sbg_ctx* ctx, float* x, float* y, float* p) {
  CHECK_CTX(ctx);
  if (!ctx->dX) return ctx->fail(SBG_ERR_STATE, "no state");
  CK(cudaSetDevice(ctx->device));
  if (int rc = csr_sync(ctx)) return rc;
  const size_t pitch = sizeof(float) * ctx->npad, w = sizeof(float) * ctx->n;
  if (x) CK(cudaMemcpy2DAsync(x, w, ctx->dX, pitch, w, ctx->R, cudaMemcpyDeviceToHost, ctx->stream));
  if (y) CK(cudaMemcpy2DAsync(y, w, ctx->dY, pitch, w, ctx->R, cudaMemcpyDeviceToHost, ctx->stream));
  if (p) CK(cudaMemcpy2DAsync(p, w, ctx->dP, pitch, w, ctx->R, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SBG_OK;
}

static int launch_resident_default(sbg_ctx* ctx, int cur, const MultiStepArgs& a, int groups, const uint32_t* ready,
                                   int* g_mode);

int sbg_advance(sbg_ctx* ctx, const sbg_params* prm, uint64_t m_begin, uint64_t m_end) {
  CHECK_CTX(ctx);
  int rc = validate_params(ctx, prm);
  if (rc) return rc;
  if (!ctx->dX || ctx->R < 1) return ctx->fail(SBG_ERR_STATE, "state not initialised");
  if (m_end > prm->steps || m_begin > m_end)
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "state already at the final step");  // engine.cpp:59
  CK(cudaSetDevice(ctx->device));
  const bool sign = is_sign_variant(prm->variant);
  const bool honours_a = prm->variant == SBG_GBSB || prm->variant == SBG_GDSB;  // engine.cpp:64 (+GdSB)
  PhaseConsts k;
  k.a = honours_a ? float(prm->a) : 0.0f;
  k.c = float(prm->c);
  k.dt = float(prm->dt);
  k.inv = 0.0f;
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (m_end == m_begin) {  // nothing to step (engine.cpp:55-110 is never called)
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    return SBG_OK;
  }
  if (ctx->kind == KIND_CSR_I8) {
    // replica-major -> spin-major (unless the last advance left the state there), B operand, M
    // steps (ping-pong); the state stays spin-major until something reads it (csr_sync)
    const int32_t n32 = int32_t(ctx->n), R32 = int32_t(ctx->R);
    const dim3 tb(32, 8);
    const dim3 tg_in(unsigned((ctx->n + 31) / 32), unsigned((ctx->R + 31) / 32));
    float* rm[3] = {ctx->dX, ctx->dY, ctx->dP};
    float* sm[3] = {ctx->dXs, ctx->dYs, ctx->dPs};
    for (int a = 0; !ctx->csr_sm_current && a < 3; ++a) {
      transpose_f32_kernel<<<tg_in, tb, 0, ctx->stream>>>(rm[a], sm[a], R32, n32, ctx->npad, ctx->rp);
      CK(cudaGetLastError());
      ++ctx->launches;
    }
    const size_t cnt = size_t(ctx->npad) * ctx->rp;
    // the operand of the current state: left in dQ[q0] by the previous advance (same kind), or
    // built here into dQ[0]
    int q0 = 0;
    if (ctx->csr_sm_current && ctx->csr_q >= 0 && (ctx->csr_q >= 2) == sign) {
      q0 = ctx->csr_q & 1;
    } else {
      if (sign)
        csr_prep_kernel<true><<<grid_for(ctx, cnt, 256), 256, 0, ctx->stream>>>(ctx->dXs, ctx->dQ[0], cnt);
      else
        csr_prep_kernel<false><<<grid_for(ctx, cnt, 256), 256, 0, ctx->stream>>>(ctx->dXs, ctx->dQ[0], cnt);
      CK(cudaGetLastError());
      ++ctx->launches;
    }
    const float* arep = (honours_a && ctx->d_arep && ctx->arep_n == ctx->R) ? ctx->d_arep : nullptr;
    // Replica slabs (SBG_CSR_SLAB = width, a multiple of 128): replicas are independent, so the M
    // steps may run slab by slab, each slab's x, y, p and operand buffers (n * W * 20 B) staying in
    // L2 across its steps. Bitwise identical for every width. Measured at C3 (N=20000, R=512):
    // 71.2 us/step in one pass, 69.5 with 256-wide slabs (twice), 78.9 with 128 (launch tails:
    // too few warp tasks per launch). Default: the widest slab >= 256 that fits ~110 MB of L2,
    // when the whole state does not.
    int64_t slab = dev_knob("SBG_CSR_SLAB");
    if (slab <= 0) {
      slab = ctx->R;
      const int64_t budget = 110ll << 20, per = ctx->n * 20;
      if (ctx->n * ctx->R * 20 > budget && m_end - m_begin >= 8) {
        const int64_t w = budget / per / CSR_RCHUNK * CSR_RCHUNK;
        if (w >= 2 * CSR_RCHUNK) slab = w;
      }
    }
    slab = std::max<int64_t>(CSR_RCHUNK, (slab + CSR_RCHUNK - 1) / CSR_RCHUNK * CSR_RCHUNK);
    // SBG_CSR_ASYNC = NB in {4, 8, 12, 16}: gathers staged through shared memory by cp.async,
    // NB per warp in flight (csr_step_async_kernel); 0 = the register-path kernel.
    const int csra = dev_knob("SBG_CSR_ASYNC");
    // SBG_CSR_LEAN: -1 = the round-1 register-path kernel, 1 / 2 / 4 = csr_step_lean_kernel with that
    // many gathers per round, unset = the default (needs 32-bit byte offsets into the operand)
    int lean = dev_knob("SBG_CSR_LEAN");
    if (lean == 0) lean = CSR_LEAN_DEFAULT;
    if (lean != -1 && lean != 1 && lean != 2 && lean != 4)
      return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "SBG_CSR_LEAN must be -1, 1, 2 or 4");
    if (lean < 0 || uint64_t(ctx->npad) * uint64_t(ctx->rp) * 4 >= (1ull << 32)) lean = 0;
    if (csra && csra != 4 && csra != 8 && csra != 12 && csra != 16)
      return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "SBG_CSR_ASYNC must be 0, 4, 8, 12 or 16");
    for (int64_t r0 = 0; r0 < ctx->R; r0 += slab) {
      const int32_t Rs = int32_t(std::min<int64_t>(slab, ctx->R - r0));
      const int64_t tasks = ctx->n * ((Rs + CSR_RCHUNK - 1) / CSR_RCHUNK);
      int blocks =
          int(std::min<int64_t>((tasks + CSR_THREADS / 32 - 1) / (CSR_THREADS / 32), int64_t(ctx->sms) * 8));
      // dev: SBG_CSR_BLOCKS = grid size of a step launch (tasks per warp = tasks / (8 * blocks))
      if (const int kb = dev_knob("SBG_CSR_BLOCKS"); kb > 0) blocks = std::min(blocks, kb);
      const size_t gsz = sign ? 1 : 4;
      const void* qa = reinterpret_cast<const char*>(ctx->dQ[q0]) + size_t(r0) * gsz;
      void* qb = reinterpret_cast<char*>(ctx->dQ[q0 ^ 1]) + size_t(r0) * gsz;
      const void* gq[2] = {qa, qb};
      float *xs = ctx->dXs + r0, *ys = ctx->dYs + r0, *ps = ctx->dPs + r0;
      const float* ar = arep ? arep + r0 : nullptr;
      int cur = 0;
      for (uint64_t m = m_begin; m < m_end; ++m) {
        PhaseConsts km = k;
        km.inv = 1.0f / static_cast<float>(prm->steps - m);  // == __frcp_rn(M - m)
        void* gn = const_cast<void*>(gq[cur ^ 1]);
        if (csra) {
          cudaError_t e = cudaErrorInvalidValue;
#define CSRA_CASE(NB)                                                                                        \
  case NB:                                                                                                   \
    e = sign ? launch_csr_async<true, NB>(ctx->stream, ctx->sms, n32, ctx->d_rowptr, ctx->d_col, ctx->d_val, \
                                          gq[cur], gn, xs, ys, ps, ctx->rp, Rs, km, ar)                      \
             : launch_csr_async<false, NB>(ctx->stream, ctx->sms, n32, ctx->d_rowptr, ctx->d_col,           \
                                           ctx->d_val, gq[cur], gn, xs, ys, ps, ctx->rp, Rs, km, ar);       \
    break;
          switch (csra) {
            CSRA_CASE(4)
            CSRA_CASE(8)
            CSRA_CASE(12)
            CSRA_CASE(16)
          }
#undef CSRA_CASE
          CK(e);
        } else if (const int pf = dev_knob("SBG_CSR_PF"); pf == 6 || pf == 7) {
          // dev: gather loop pipelined by one (two gathers in flight per warp), pf blocks per SM
          const int pblocks = int(std::min<int64_t>((tasks + CSR_THREADS / 32 - 1) / (CSR_THREADS / 32),
                                                    int64_t(ctx->sms) * pf));
#define CSR_PF(S, B) \
  csr_step_pf_kernel<S, B><<<pblocks, CSR_THREADS, 0, ctx->stream>>>(n32, ctx->d_rowptr, ctx->d_col, ctx->d_val, \
                                                                   gq[cur], gn, xs, ys, ps, ctx->rp, Rs, km, ar)
          if (sign) {
            if (pf == 6) CSR_PF(true, 6); else CSR_PF(true, 7);
          } else {
            if (pf == 6) CSR_PF(false, 6); else CSR_PF(false, 7);
          }
#undef CSR_PF
        } else if (lean) {
          // fewer instructions per task (csr_step_lean_kernel), `lean` nonzeros per gather round
          const PhaseIdent ident{-0.0f, 1.0f, -1.0f};
          const bool pfs = dev_knob("SBG_CSR_PFS") == 1;  // x, y, p prefetched into shared memory by cp.async
#define CSR_LEAN(S, U)                                                                                          \
  (pfs ? csr_step_lean_kernel<S, U, true> : csr_step_lean_kernel<S, U, false>)<<<blocks, CSR_THREADS, 0, ctx->stream>>>( \
      uint32_t(n32), ctx->d_rowptr, ctx->d_col, ctx->d_val, gq[cur], gn, xs, ys, ps, uint32_t(ctx->rp), uint32_t(Rs),  \
      km, ident, ar)
          if (sign) {
            if (lean == 1) CSR_LEAN(true, 1); else if (lean == 2) CSR_LEAN(true, 2); else CSR_LEAN(true, 4);
          } else {
            if (lean == 1) CSR_LEAN(false, 1); else if (lean == 2) CSR_LEAN(false, 2); else CSR_LEAN(false, 4);
          }
#undef CSR_LEAN
        } else if (sign)
          csr_step_sm_kernel<true><<<blocks, CSR_THREADS, 0, ctx->stream>>>(
              n32, ctx->d_rowptr, ctx->d_col, ctx->d_val, gq[cur], gn, xs, ys, ps, ctx->rp, Rs, km, ar);
        else
          csr_step_sm_kernel<false><<<blocks, CSR_THREADS, 0, ctx->stream>>>(
              n32, ctx->d_rowptr, ctx->d_col, ctx->d_val, gq[cur], gn, xs, ys, ps, ctx->rp, Rs, km, ar);
        CK(cudaGetLastError());
        ++ctx->launches;
        cur ^= 1;
      }
    }
    ctx->csr_sm_current = true;
    ctx->csr_q = (q0 ^ int((m_end - m_begin) & 1)) + (sign ? 2 : 0);
  } else {
    const bool resident = use_resident(ctx, prm->variant);
    const int knob = dev_knob("SBG_STEP_CFG");
    const bool pair_ok = (ctx->npad % 256) == 0;
    // streaming sign launches on e2m1 operands (the J-streaming regime, e.g. C5: half the bytes)
    const bool q4s = sign && !resident && q4_stream(ctx);
    const int need = q4s ? 2 : sign ? 1 : NPL;
    if (ctx->g_mode != need && !resident) {  // the resident kernel publishes its own G_0
      if (q4s) {
        const size_t tot = size_t(ctx->rpad) * (ctx->npad / 2);
        prep_sign4_kernel<<<grid_for(ctx, tot, 256), 256, 0, ctx->stream>>>(
            ctx->dX, ctx->dG[ctx->g_cur], int32_t(ctx->n), int32_t(ctx->npad), int32_t(ctx->R), int32_t(ctx->rpad),
            gdim(ctx) / 2, ctx->sharded ? ctx->row0 : 0);
        CK(cudaGetLastError());
        ++ctx->launches;
      } else {
        rc = prep_planes(ctx, ctx->dX, ctx->dG[ctx->g_cur], need, ctx->R, ctx->rpad, /*into_global=*/true);
        if (rc) return rc;
      }
      ctx->g_mode = need;
    }
    if (resident) ctx->g_mode = 1;
    const bool fx = ctx->kind == KIND_DENSE_FX;
    // real J x 4 x-planes: 64-replica tiles with one accumulator buffer (6 x 64 TMEM columns)
    // halve the MMA instruction count of 32-replica tiles; SBG_FX_BN=32 selects the latter
    const bool fx64 = fx && !sign && dev_knob("SBG_FX_BN") != 32;
    const int bn = fx64 ? BN_FX_PLANE_W : fx ? (sign ? BN_FX_SIGN : BN_FX_PLANE) : (sign ? BN_SIGN : BN_PLANE);
    const int64_t T = (ctx->npad / 128) * (ctx->rpad / bn);
    const int64_t max_steps = std::max<int64_t>(1, (int64_t(1) << 30) / T);
    const bool per_step = dev_knob("SBG_PER_STEP_LAUNCH") != 0;
    for (uint64_t m = m_begin; m < m_end;) {
      const int64_t ns = per_step ? 1 : std::min<int64_t>(int64_t(m_end - m), max_steps);
      MultiStepArgs a;
      std::memset(&a, 0, sizeof a);
      a.n = int32_t(ctx->n);
      a.npad = int32_t(ctx->npad);
      a.R = int32_t(ctx->R);
      a.rpad = int32_t(ctx->rpad);
      a.num_m = int32_t(ctx->npad / 128);
      a.num_n = int32_t(ctx->rpad / bn);
      a.fx_exp = sign ? -ctx->fx_shift : -(ctx->fx_shift + 30);
      a.k = k;
      a.M = prm->steps;
      a.t_begin = m;
      a.nsteps = int32_t(ns);
      a.done = ctx->d_done;
      a.a_rep = (honours_a && ctx->d_arep && ctx->arep_n == ctx->R) ? ctx->d_arep : nullptr;
      a.sx = ctx->dX;
      a.sy = ctx->dY;
      a.sp = ctx->dP;
      const int cur = ctx->g_cur;
      a.kpad = int32_t(ctx->sharded ? ctx->kpad : ctx->npad);
      a.num_m_total = int32_t(ctx->sharded ? ctx->num_m_total : ctx->npad / 128);
      a.col0 = int32_t(ctx->sharded ? ctx->row0 : 0);
      a.done_base = ctx->sharded ? ctx->done_base : 0;
      a.g_ld = (ctx->sharded ? ctx->kpad : ctx->npad) / (q4s ? 2 : 1);  // bytes per G row
      a.npeers = ctx->sharded ? int32_t(ctx->peer_done.size()) : 0;
      a.err = ctx->d_err;
      for (int pr = 0; pr < a.npeers; ++pr) {
        // step parity 0 writes buffer cur^1, parity 1 buffer cur (as the local Gout maps)
        a.peer_g[0][pr] = cur == 0 ? ctx->peer_g1[size_t(pr)] : ctx->peer_g0[size_t(pr)];
        a.peer_g[1][pr] = cur == 0 ? ctx->peer_g0[size_t(pr)] : ctx->peer_g1[size_t(pr)];
        a.peer_done[pr] = ctx->peer_done[size_t(pr)];
      }
      a.dbg = hook_knob("SBG_STEP_DBG");
      // Defaults (measured on B200, tools/step_driver.py): sign variants on CTA pairs
      // (3 operand stages, 4 state buffers): 73 us/step at N=2000, R=8192, vs 83 us
      // single-CTA; fixed-point planes single-CTA (3, 2): 18.5 us/step at R=1024 vs
      // 20.4 us on pairs. SBG_STEP_CFG selects sweep alternatives (dev only).
      if (fx) {
        // real-valued J: 3 J planes x (sign | 4 x-planes), single-CTA
#if SBG_FX_BK == 64
        // dev: 64-byte K stages, 4 deep (bitwise equal, measured slower: DESIGN K4)
        TmaMaps mq = fx64 ? ctx->fxq_planes64[cur] : ctx->fxq_planes32[cur];
        mq.J = ctx->tmJfx64;
        rc = sign   ? launch_multistep<1, BN_FX_SIGN, 2, 4, FX_NA>(ctx, ctx->fxmaps_sign[cur], a)
             : fx64 ? launch_multistep<NPL, BN_FX_PLANE_W, 4, 2, FX_NA>(ctx, mq, a)
                    : launch_multistep<NPL, BN_FX_PLANE, 4, 3, FX_NA>(ctx, mq, a);
#else
        // continuous variants on CTA pairs (128-replica pair tiles, nine products, one
        // accumulator buffer); SBG_FX_PAIR=0 selects the single-CTA kernel (dev comparison)
        if (!sign && fx64 && !getenv_is0("SBG_FX_PAIR") && ctx->rpad % 128 == 0 && (ctx->npad / 128) % 2 == 0)
          rc = launch_multistep_pair<NPL, 128, 2, 2, 16, false, FX_NA>(ctx, ctx->maps_planes[cur], a);
        else
          rc = sign   ? launch_multistep<1, BN_FX_SIGN, 2, 4, FX_NA>(ctx, ctx->fxmaps_sign[cur], a)
               : fx64 ? launch_multistep<NPL, BN_FX_PLANE_W, 2, 2, FX_NA>(ctx, ctx->maps_planes[cur], a)
                      : launch_multistep<NPL, BN_FX_PLANE, 2, 3, FX_NA>(ctx, ctx->fxmaps_planes[cur], a);
#endif
      } else if (resident) {
        // default for sign variants: state resident in TMEM (step_resident.cuh); SBG_RESIDENT=0
        // selects the streaming kernels (dev comparison)
        switch (dev_knob("SBG_RES_CFG")) {
          case 1: rc = launch_resident<16, 8>(ctx, ctx->rmaps_sign[cur], a); break;
          case 2: rc = launch_resident<8, 8>(ctx, ctx->rmaps_sign[cur], a); break;
          case 3: rc = launch_resident<8, 4>(ctx, ctx->rmaps_sign[cur], a); break;
          case 6: rc = launch_resident<16, 4, 6>(ctx, ctx->rmaps_sign[cur], a); break;
          case 7: rc = launch_resident<16, 4, 7>(ctx, ctx->rmaps_sign[cur], a); break;
          case 11: rc = launch_resident<16, 4>(ctx, ctx->rmaps_sign[cur], a); break;  // NR 128, all in TMEM
          case 12: rc = launch_resident<16, 4, RES_NR_STAGES, RES_NR>(ctx, ctx->rmaps160_sign[cur], a); break;
          default: {
            int gm = 1;
            rc = launch_resident_default(ctx, cur, a, -1, nullptr, &gm);
            ctx->g_mode = gm;
          }
        }
      } else if (sign) {
        switch (pair_ok ? knob : -1) {
          case -1: rc = launch_multistep<1, BN_SIGN, SIGN_STAGES, SIGN_NBUF>(ctx, ctx->maps_sign[cur], a); break;
          case 2: rc = launch_multistep_pair<1, NPAIR_SIGN, 2, 6>(ctx, ctx->maps_sign[cur], a); break;
          case 3: rc = launch_multistep_pair<1, NPAIR_SIGN, 4, 3>(ctx, ctx->maps_sign[cur], a); break;
          case 4: rc = launch_multistep_pair<1, NPAIR_SIGN, 2, 5>(ctx, ctx->maps_sign[cur], a); break;
          case 5: rc = launch_multistep_pair<1, NPAIR_SIGN, 3, 8, 8>(ctx, ctx->maps_sign_cw8[cur], a); break;
          case 6: rc = launch_multistep_pair<1, NPAIR_SIGN, 2, 10, 8>(ctx, ctx->maps_sign_cw8[cur], a); break;
          case 7: rc = launch_multistep_pair<1, NPAIR_SIGN, 5, 2>(ctx, ctx->maps_sign[cur], a); break;
          case 8: rc = launch_multistep_pair<1, NPAIR_SIGN, 3, 4>(ctx, ctx->maps_sign[cur], a); break;
          // non-resident sign launches are the large-N J-streaming regime (C5: 2.06 ms/step,
          // 0.79 of HBM with 5 operand stages vs 2.29 ms with 3); e2m1 operands halve J
          default:
            if (q4s)
              tail_split(ctx, (ctx->npad / 256) * (ctx->rpad / NPAIR_SIGN), a);
            else
              a.ksplit = 1;
            if (q4s && q4_narrow(ctx)) {
              a.n_fast = 1;
              rc = launch_multistep_pair<1, 128, 5, 2, 16, true>(ctx, ctx->pq128maps_sign[cur], a);
            } else {
              const int c5 = dev_knob("SBG_C5_CFG");  // dev: (operand stages, state buffers) alternatives
              if (q4s && c5 == 43)
                rc = launch_multistep_pair<1, NPAIR_SIGN, 4, 3, 16, true>(ctx, ctx->pqmaps_sign[cur], a);
              else if (q4s && c5 == 34)
                rc = launch_multistep_pair<1, NPAIR_SIGN, 3, 4, 16, true>(ctx, ctx->pqmaps_sign[cur], a);
              else
                rc = q4s ? launch_multistep_pair<1, NPAIR_SIGN, 5, 2, 16, true>(ctx, ctx->pqmaps_sign[cur], a)
                         : launch_multistep_pair<1, NPAIR_SIGN, 5, 2>(ctx, ctx->maps_sign[cur], a);
            }
        }
      } else {
        switch (pair_ok ? knob : -1) {
          case 2: rc = launch_multistep_pair<NPL, NPAIR_PLANE, 3, 3>(ctx, ctx->pmaps_planes[cur], a); break;
          case 3: rc = launch_multistep_pair<NPL, NPAIR_PLANE, 4, 2>(ctx, ctx->pmaps_planes[cur], a); break;
          case 6: rc = launch_multistep_pair<NPL, NPAIR_PLANE, 5, 2>(ctx, ctx->pmaps_planes[cur], a); break;
          // 128-replica pair tiles, one accumulator buffer (B halves of 64 rows: the maps_planes boxes)
          case 9: rc = launch_multistep_pair<NPL, 2 * BN_PLANE, 3, 2>(ctx, ctx->maps_planes[cur], a); break;
          case 7: rc = launch_multistep<NPL, BN_PLANE, PLANE_STAGES, PLANE_NBUF>(ctx, ctx->maps_planes[cur], a); break;
          case 4: {  // smaller replica tiles: more tiles per step for small R
            MultiStepArgs a32 = a;
            a32.num_n = int32_t(ctx->rpad / 32);
            rc = launch_multistep<NPL, 32, 4, 3>(ctx, ctx->fxmaps_planes[cur], a32);
            break;
          }
          case 5: {
            MultiStepArgs a32 = a;
            a32.num_n = int32_t(ctx->rpad / 32);
            rc = launch_multistep<NPL, 32, 3, 4>(ctx, ctx->fxmaps_planes[cur], a32);
            break;
          }
          default: {
            // 128-replica tiles halve the MMA instructions per output but only pay with enough
            // tiles per step to fill the pairs (>= 2.5 waves; measured at n = 2000, GbSB:
            // R = 3072 46.7 -> 43.9 us/step, R = 8192 132.1 -> 127.5; R = 1000 15.1 -> 23.5)
            const int64_t wide_tiles = (ctx->npad / 256) * (ctx->rpad / (2 * BN_PLANE));
            if (2 * wide_tiles >= 5 * int64_t(ctx->sms / 2))
              rc = launch_multistep_pair<NPL, 2 * BN_PLANE, 3, 2>(ctx, ctx->maps_planes[cur], a);
            else
              rc = launch_multistep_pair<NPL, NPAIR_PLANE, 4, 2>(ctx, ctx->pmaps_planes[cur], a);
          }
        }
      }
      if (rc) return rc;
      ctx->g_cur = cur ^ int(ns & 1);
      m += uint64_t(ns);
    }
  }
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  return SBG_OK;
}

double sbg_last_advance_ms(const sbg_ctx* ctx) {
  if (!ctx) return -1.0;
  cudaSetDevice(ctx->device);
  if (cudaEventSynchronize(ctx->ev[1]) != cudaSuccess) return -1.0;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]) != cudaSuccess) return -1.0;
  return ms;
}

namespace {
// Energies of every replica (device) + argmin; leaves dE2/dBest/dSign populated.
int readout_device(sbg_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  int rc = csr_sync(ctx);
  if (rc) return rc;
  CK(cudaMemsetAsync(ctx->dE2, 0, sizeof(unsigned long long) * ctx->rpad, ctx->stream));
  if (ctx->kind == KIND_CSR_I8) {
    rc = launch_csr_readout(ctx->stream, ctx->sms, int32_t(ctx->n), ctx->d_rowptr, ctx->d_col, ctx->d_val,
                            ctx->dX, ctx->npad, int32_t(ctx->R), ctx->dSign, ctx->dE2);
    if (rc) return ctx->fail(SBG_ERR_CUDA, "CSR readout failed: %s", cudaGetErrorString(cudaError_t(rc)));
    ctx->launches += 1;
  } else {
    rc = prep_planes(ctx, ctx->dX, ctx->dSign, 1, ctx->R, ctx->rpad);
    if (rc) return rc;
    StepArgs a = base_args(ctx, BN_SIGN, ctx->R, ctx->rpad);
    a.sign_in = reinterpret_cast<const int8_t*>(ctx->dSign);
    if (ctx->kind == KIND_DENSE_FX) {
      // E2 = sum_a 2^(8a) E2_a over the J byte planes (u8, u8, s8), exact in int64
      CK(cudaMemsetAsync(ctx->dE2p, 0, sizeof(unsigned long long) * ctx->rpad * FX_NA, ctx->stream));
      for (int pa = 0; pa < FX_NA; ++pa) {
        a.e2 = ctx->dE2p + size_t(pa) * ctx->rpad;
        a.a_unsigned = pa < FX_NA - 1;
        rc = launch_step<1, BN_SIGN, EpiMode::Readout>(ctx, ctx->tmSign, a, &ctx->tmJplane[pa]);
        if (rc) return rc;
      }
      combine_planes_e2_kernel<<<grid_for(ctx, size_t(ctx->R), 256), 256, 0, ctx->stream>>>(
          reinterpret_cast<const long long*>(ctx->dE2p), ctx->rpad, FX_NA, int32_t(ctx->R),
          reinterpret_cast<long long*>(ctx->dE2));
      CK(cudaGetLastError());
      ++ctx->launches;
    } else {
      a.e2 = ctx->dE2;
      rc = launch_step<1, BN_SIGN, EpiMode::Readout>(ctx, ctx->tmSign, a);
      if (rc) return rc;
    }
  }
  argmin_energy_kernel<<<1, 1024, 0, ctx->stream>>>(reinterpret_cast<const long long*>(ctx->dE2),
                                                    int32_t(ctx->R), ctx->dBest);
  CK(cudaGetLastError());
  ++ctx->launches;
  return SBG_OK;
}
}  // namespace

int sbg_readout(sbg_ctx* ctx, int8_t* spins, double* energy, int64_t* best_index, double* best_energy) {
  CHECK_CTX(ctx);
  if (!ctx->dX || ctx->R < 1) return ctx->fail(SBG_ERR_STATE, "state not initialised");
  int rc = readout_device(ctx);
  if (rc) return rc;
  if (spins)
    CK(cudaMemcpy2DAsync(spins, ctx->n, ctx->dSign, ctx->npad, ctx->n, ctx->R, cudaMemcpyDeviceToHost,
                         ctx->stream));
  std::vector<long long> e2;
  if (energy) {
    e2.resize(ctx->R);
    CK(cudaMemcpyAsync(e2.data(), ctx->dE2, sizeof(long long) * ctx->R, cudaMemcpyDeviceToHost, ctx->stream));
  }
  long long best[2] = {0, 0};
  CK(cudaMemcpyAsync(best, ctx->dBest, sizeof best, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  // ising_energy = -1/2 sum_i s_i (J s)_i, exact in double for integer J
  if (energy)
    for (int64_t r = 0; r < ctx->R; ++r) energy[r] = -0.5 * double(e2[size_t(r)]) * ctx->energy_scale;
  if (best_index) *best_index = best[0];
  if (best_energy) *best_energy = -0.5 * double(best[1]) * ctx->energy_scale;
  return SBG_OK;
}

int sbg_readout_best(sbg_ctx* ctx, int8_t* best_spins, double* best_energy, int64_t* best_index, double* energies) {
  CHECK_CTX(ctx);
  if (!ctx->dX || ctx->R < 1) return ctx->fail(SBG_ERR_STATE, "state not initialised");
  int rc = readout_device(ctx);
  if (rc) return rc;
  long long best[2] = {0, 0};
  CK(cudaMemcpyAsync(best, ctx->dBest, sizeof best, cudaMemcpyDeviceToHost, ctx->stream));
  std::vector<long long> e2;
  if (energies) {
    e2.resize(ctx->R);
    CK(cudaMemcpyAsync(e2.data(), ctx->dE2, sizeof(long long) * ctx->R, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  if (best_spins)
    CK(cudaMemcpy(best_spins, ctx->dSign + size_t(best[0]) * ctx->npad, ctx->n, cudaMemcpyDeviceToHost));
  if (energies)
    for (int64_t r = 0; r < ctx->R; ++r) energies[r] = -0.5 * double(e2[size_t(r)]) * ctx->energy_scale;
  if (best_index) *best_index = best[0];
  if (best_energy) *best_energy = -0.5 * double(best[1]) * ctx->energy_scale;
  return SBG_OK;
}

int sbg_fields_sign(sbg_ctx* ctx, int64_t R, const int8_t* S, int32_t* F) {
  CHECK_CTX(ctx);
  if (ctx->kind != KIND_DENSE_I8) return ctx->fail(SBG_ERR_STATE, "dense couplings not set");
  if (R < 1 || !S || !F) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  const int64_t rpad = round_up(R, PAD_R);
  const size_t pl = size_t(rpad) * ctx->npad;
  int8_t* dS = nullptr;
  uint8_t* dGs = nullptr;
  int32_t* dF = nullptr;
  CK(cudaMalloc(&dS, size_t(R) * ctx->n));
  CK(cudaMalloc(&dGs, pl));
  CK(cudaMalloc(&dF, sizeof(int32_t) * pl));
  CK(cudaMemcpyAsync(dS, S, size_t(R) * ctx->n, cudaMemcpyHostToDevice, ctx->stream));
  pad_plane_kernel<<<grid_for(ctx, pl, 256), 256, 0, ctx->stream>>>(dS, dGs, int32_t(ctx->n),
                                                                    int32_t(ctx->npad), int32_t(R), int32_t(rpad));
  CK(cudaGetLastError());
  CUtensorMap tm;
  int rc = encode_2d_u8(ctx, &tm, dGs, ctx->npad, rpad, 128, BN_SIGN);
  if (rc == SBG_OK) {
    StepArgs a = base_args(ctx, BN_SIGN, R, rpad);
    a.fields_out = dF;
    rc = launch_step<1, BN_SIGN, EpiMode::Fields>(ctx, tm, a);
  }
  if (rc == SBG_OK) {
    CK(cudaMemcpy2DAsync(F, sizeof(int32_t) * ctx->n, dF, sizeof(int32_t) * ctx->npad, sizeof(int32_t) * ctx->n,
                         R, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  cudaFree(dS);
  cudaFree(dGs);
  cudaFree(dF);
  return rc;
}

int sbg_fields_fixed(sbg_ctx* ctx, int64_t R, const float* x, float* F) {
  CHECK_CTX(ctx);
  if (ctx->kind != KIND_DENSE_I8) return ctx->fail(SBG_ERR_STATE, "dense couplings not set");
  if (R < 1 || !x || !F) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  const int64_t rpad = round_up(R, PAD_R);
  const size_t pl = size_t(rpad) * ctx->npad;
  float* dx = nullptr;
  uint8_t* dGp = nullptr;
  float* dF = nullptr;
  CK(cudaMalloc(&dx, sizeof(float) * pl));
  CK(cudaMalloc(&dGp, NPL * pl));
  CK(cudaMalloc(&dF, sizeof(float) * pl));
  CK(cudaMemsetAsync(dx, 0, sizeof(float) * pl, ctx->stream));
  CK(cudaMemcpy2DAsync(dx, sizeof(float) * ctx->npad, x, sizeof(float) * ctx->n, sizeof(float) * ctx->n, R,
                       cudaMemcpyHostToDevice, ctx->stream));
  int rc = prep_planes(ctx, dx, dGp, NPL, R, rpad);
  CUtensorMap tm;
  if (rc == SBG_OK) rc = encode_2d_u8(ctx, &tm, dGp, ctx->npad, NPL * rpad, 128, BN_PLANE);
  if (rc == SBG_OK) {
    StepArgs a = base_args(ctx, BN_PLANE, R, rpad);
    a.fields_out = dF;
    rc = launch_step<NPL, BN_PLANE, EpiMode::Fields>(ctx, tm, a);
  }
  if (rc == SBG_OK) {
    CK(cudaMemcpy2DAsync(F, sizeof(float) * ctx->n, dF, sizeof(float) * ctx->npad, sizeof(float) * ctx->n, R,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  cudaFree(dx);
  cudaFree(dGp);
  cudaFree(dF);
  return rc;
}

static int run_tail(sbg_ctx* ctx, const sbg_params* prm, float* x_final, int8_t* spins, double* energy,
                    int64_t* best_index, sbg_timing* timing, bool advanced = false) {
  int rc;
  if (!advanced) {
    CK(cudaEventRecord(ctx->ev[3], ctx->stream));
    rc = sbg_advance(ctx, prm, 0, prm->steps);
    if (rc) return rc;
  }
  CK(cudaEventRecord(ctx->ev[4], ctx->stream));
  rc = spins ? sbg_readout(ctx, spins, energy, best_index, nullptr)
             : sbg_readout_best(ctx, ctx->tail_best_spins, ctx->tail_best_energy, best_index, energy);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev[5], ctx->stream));
  if (x_final) {
    const size_t pitch = sizeof(float) * ctx->npad, w = sizeof(float) * ctx->n;
    if (int rc2 = csr_sync(ctx)) return rc2;
    CK(cudaMemcpy2DAsync(x_final, w, ctx->dX, pitch, w, ctx->R, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaEventRecord(ctx->ev[6], ctx->stream));
  CK(cudaEventSynchronize(ctx->ev[6]));
  if (timing) {
    float a = 0, b = 0, c = 0, d = 0, e = 0;
    cudaEventElapsedTime(&a, ctx->ev[2], ctx->ev[7]);
    cudaEventElapsedTime(&b, ctx->ev[7], ctx->ev[3]);
    cudaEventElapsedTime(&c, ctx->ev[3], ctx->ev[4]);
    cudaEventElapsedTime(&d, ctx->ev[4], ctx->ev[5]);
    cudaEventElapsedTime(&e, ctx->ev[5], ctx->ev[6]);
    timing->h2d_ms = a;
    timing->init_ms = b;
    timing->steps_ms = c;
    timing->readout_ms = d;
    timing->d2h_ms = e;
    timing->total_ms = a + b + c + d + e;
    timing->kernel_launches = ctx->launches;
  }
  return SBG_OK;
}

// Tensor maps of the parts kernel for G-buffer parity cur and part widths w0 (class 0), w1 (class 1).
static int encode_part_maps(sbg_ctx* ctx, PartMaps* pm, int cur, int w0, int w1) {
  pm->J = ctx->tmJ4;
  const uint64_t gb = uint64_t(ctx->npad / 2), gv4 = uint64_t((ctx->n + 1) / 2);
  const int ws[2] = {w0, w1};
  auto enc = get_encode();
  if (!enc) return ctx->fail(SBG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  const uint32_t kbs = uint32_t(std::min<int64_t>(8, ctx->npad / 256));  // K blocks (J resident: <= 8)
  for (int c = 0; c < 2; ++c)
    for (int par = 0; par < 2; ++par) {
      // [K block][rpad][128 B] view of G (K block kb = bytes [128 kb, 128 kb + 128) of each row)
      cuuint64_t dims[3] = {128, cuuint64_t(ctx->rpad), cuuint64_t(gb / 128)};
      cuuint64_t strides[2] = {cuuint64_t(gb), 128};
      cuuint32_t box[3] = {128, uint32_t(ws[c] / 2), kbs}, es[3] = {1, 1, 1};
      if (enc(&pm->Gin3[c][par], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ctx->dG[cur ^ par], dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return ctx->fail(SBG_ERR_CUDA, "cuTensorMapEncodeTiled (3D G) failed");
      int rc = encode_2d_u8(ctx, &pm->Gin[c][par], ctx->dG[cur ^ par], gb, uint64_t(ctx->rpad), 128, uint32_t(ws[c] / 2));
      if (!rc)
        rc = encode_2d(ctx, &pm->Gout[c][par], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ctx->dG[cur ^ par ^ 1], gv4,
                       uint64_t(ctx->R), gb, 64, uint32_t(ws[c]), CU_TENSOR_MAP_SWIZZLE_NONE);
      if (rc) return rc;
    }
  return SBG_OK;
}

extern "C++" {
// The TS kernel (J in TMEM, x, y in shared memory): the parts kernel's G maps plus 2D boxes
// {128 spins, 160 replicas} of the replica-major x and y (rows >= rpad read as zero).
template <int PARTS, int ST, bool PKB, bool KH2 = false>
int launch_ts(sbg_ctx* ctx, int cur, const MultiStepArgs& a, int groups, const uint32_t* ready) {
  using T = PartTable<PARTS>;
  TsMapKey key;
  key.g0 = ctx->dG[0];
  key.g1 = ctx->dG[1];
  key.x = ctx->dX;
  key.y = ctx->dY;
  key.j4 = ctx->dJ4;
  key.n = ctx->n;
  key.npad = ctx->npad;
  key.R = ctx->R;
  key.rpad = ctx->rpad;
  key.w0 = T::W[0];
  key.w1 = T::W[PARTS - 1];
  if (!KH2 && ctx->ts_ok[cur] && ctx->ts_key[cur] == key) {
    if (a.nsteps < 1) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "resident launch without steps");
    return launch_resident<16, 4, ST, RES_NR, true, -PARTS, true, TsMaps, PKB, KH2>(ctx, ctx->ts_cache[cur], a, 0,
                                                                                     groups, ready);
  }
  ctx->ts_ok[cur] = false;
  TsMaps tm;
  int rc = encode_part_maps(ctx, &tm.g, cur, T::W[0], T::W[PARTS - 1]);
  if (rc) return rc;
  if (KH2) {  // the 3D G view with box depth KB / 2
    auto enc = get_encode();
    const uint64_t gb = uint64_t(ctx->npad / 2);
    const uint32_t kh = uint32_t(ctx->npad / 512);
    const int ws2[2] = {T::W[0], T::W[PARTS - 1]};
    for (int c = 0; c < 2; ++c)
      for (int par = 0; par < 2; ++par) {
        cuuint64_t dims[3] = {128, cuuint64_t(ctx->rpad), cuuint64_t(gb / 128)};
        cuuint64_t strides[2] = {cuuint64_t(gb), 128};
        cuuint32_t box[3] = {128, uint32_t(ws2[c] / 2), kh}, es[3] = {1, 1, 1};
        if (enc(&tm.Gin3h[c][par], CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ctx->dG[cur ^ par], dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return ctx->fail(SBG_ERR_CUDA, "cuTensorMapEncodeTiled (3D G halves) failed");
      }
  }
  const int ws[2] = {T::W[0], T::W[PARTS - 1]};
  for (int c = 0; c < 2 && !rc; ++c) {
    rc = encode_2d(ctx, &tm.X[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ctx->dX, uint64_t(ctx->npad),
                   uint64_t(ctx->rpad), sizeof(float) * ctx->npad, 128, uint32_t(ws[c]), CU_TENSOR_MAP_SWIZZLE_NONE);
    if (!rc)
      rc = encode_2d(ctx, &tm.Y[c], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ctx->dY, uint64_t(ctx->npad),
                     uint64_t(ctx->rpad), sizeof(float) * ctx->npad, 128, uint32_t(ws[c]), CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  if (rc) return rc;
  if (!KH2) {
    ctx->ts_cache[cur] = tm;
    ctx->ts_key[cur] = key;
    ctx->ts_ok[cur] = true;
    // the other G-buffer parity too (an odd-length advance flips it): the next launch hits
    TsMaps other = tm;
    rc = encode_part_maps(ctx, &other.g, cur ^ 1, T::W[0], T::W[PARTS - 1]);
    if (rc) return rc;
    ctx->ts_cache[cur ^ 1] = other;
    ctx->ts_key[cur ^ 1] = key;
    ctx->ts_ok[cur ^ 1] = true;
  }
  if (a.nsteps < 1) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "resident launch without steps");
  return launch_resident<16, 4, ST, RES_NR, true, -PARTS, true, TsMaps, PKB, KH2>(ctx, tm, a, 0, groups, ready);
}

template <int PARTS, int ST, bool JRES>
int launch_parts(sbg_ctx* ctx, int cur, const MultiStepArgs& a, int groups, const uint32_t* ready) {
  using T = PartTable<PARTS>;
  PartMaps pm;
  const int rc = encode_part_maps(ctx, &pm, cur, T::W[0], T::W[PARTS - 1]);
  if (rc) return rc;
  return launch_resident<16, 4, ST, RES_NR, true, PARTS, JRES>(ctx, pm, a, 0, groups, ready);
}
}

// The default resident launch: NR 160 when it cuts the group count, e2m1 operands when J
// has an e2m1 copy. Returns the G-buffer mode left behind (1 = int8 sign plane, 0 = e2m1).
static int launch_resident_default(sbg_ctx* ctx, int cur, const MultiStepArgs& a, int groups, const uint32_t* ready,
                                   int* g_mode) {
  const bool q4 = ctx->dJ4 != nullptr && !ctx->sharded;
  *g_mode = q4 ? 0 : 1;
  if (resident_nr(ctx) == RES_NR) {
    // e2m1: the parts kernel, PARTS interleaved column-part chains (SBG_RES_SPLIT=0 = one chain,
    // SBG_RES_PARTS=2/3: fewer, wider parts, dev). npad <= 2048: J resident in shared memory and
    // each part-step's G in one 3D TMA load; larger npad: 2 parts, J streamed.
    if (q4 && !getenv_is0("SBG_RES_SPLIT")) {
      if (ctx->npad > 2048) return launch_parts<2, 10, false>(ctx, cur, a, groups, ready);
      // default: J in TMEM (TS MMAs at the N/2 floor), x, y in shared memory; SBG_RES_TS=0: the
      // parts kernel (J in shared memory)
      if (!getenv_is0("SBG_RES_TS")) {
        // (wider parts' G super-stages do not fit beside x and y in shared memory)
        // SBG_RES_PKB=1 (dev): per-K-block dependencies and MMA issue in landing order. Bitwise
        // equal, measured slower (26.7 -> 34.7 us/step): the producer's eight diverged polling
        // lanes (each acquire invalidates L1) and the MMA warp's per-part poll over all eight
        // K blocks serialise more than the wait for the slowest producer they were to hide.
        const bool pkb = dev_knob("SBG_RES_PKB") == 1;
        if (dev_knob("SBG_RES_PARTS") == 5)
          return pkb ? launch_ts<5, 3, true>(ctx, cur, a, groups, ready) : launch_ts<5, 3, false>(ctx, cur, a, groups, ready);
        // SBG_RES_KH2=1: each part-step's G in two halves (MMAs on the first while the second lands)
        if (!pkb && dev_knob("SBG_RES_KH2") == 1 && (ctx->npad / 256) % 2 == 0)
          return launch_ts<4, 2, false, true>(ctx, cur, a, groups, ready);
        return pkb ? launch_ts<4, 2, true>(ctx, cur, a, groups, ready) : launch_ts<4, 2, false>(ctx, cur, a, groups, ready);
      }
      switch (dev_knob("SBG_RES_PARTS")) {
        case 2: return launch_parts<2, 2, true>(ctx, cur, a, groups, ready);
        case 3: return launch_parts<3, 2, true>(ctx, cur, a, groups, ready);
        default: return launch_parts<4, 3, true>(ctx, cur, a, groups, ready);  // C2: 28.3 us (3: 28.3, 2: 28.9)
      }
    }
    return q4 ? launch_resident<16, 4, RES_NR_STAGES, RES_NR, true>(ctx, ctx->qmaps160_sign[cur], a, 0, groups, ready)
              : launch_resident<16, 4, RES_NR_STAGES, RES_NR>(ctx, ctx->rmaps160_sign[cur], a, 0, groups, ready);
  }
  return q4 ? launch_resident<16, 4, RES_STAGES, 128, true>(ctx, ctx->qmaps_sign[cur], a, 0, groups, ready)
            : launch_resident<16, 4>(ctx, ctx->rmaps_sign[cur], a, 0, groups, ready);
}

// sbg_run on the resident kernel: the replica blocks are independent for the whole run,
// so a block's M steps start as soon as ITS x0/y0 rows have arrived; the copies of later
// groups (copy stream) overlap the earlier groups' steps. The first group's blocks get a
// flag each (their copies are the only exposed ones), later groups one flag per group.
static int run_pipelined(sbg_ctx* ctx, const sbg_params* prm, int64_t R, const float* x0, const float* y0,
                         float* x_final, int8_t* spins, double* energy, int64_t* best_index, sbg_timing* timing) {
  int rc;
  auto write_value = get_write_value32();
  int rbg = 0, groups = 0;
  const int nr = resident_nr(ctx);
  resident_geometry(ctx, ctx->npad, ctx->rpad, &rbg, &groups, nr);
  if (!write_value || groups < 2) {  // nothing to overlap: plain path
    rc = sbg_set_state(ctx, R, x0, y0, nullptr);
    if (rc) return rc;
    CK(cudaEventRecord(ctx->ev[7], ctx->stream));
    return run_tail(ctx, prm, x_final, spins, energy, best_index, timing);
  }
  const int nflags = rbg + groups - 1;  // [0, rbg): group 0's blocks; rbg + g - 1: group g >= 1
  if (ctx->ready_cap < nflags) {
    cudaFree(ctx->d_ready);
    ctx->d_ready = nullptr;
    CK(cudaMalloc(&ctx->d_ready, sizeof(uint32_t) * nflags));
    ctx->ready_cap = nflags;
  }
  CK(cudaMemsetAsync(ctx->d_ready, 0, sizeof(uint32_t) * nflags, ctx->stream));
  const size_t cnt = size_t(ctx->rpad) * ctx->npad;
  fill_f32_kernel<<<grid_for(ctx, cnt, 256), 256, 0, ctx->stream>>>(ctx->dP, cnt, 1.0f);
  CK(cudaGetLastError());
  ++ctx->launches;
  const size_t pitch = sizeof(float) * ctx->npad, w = sizeof(float) * ctx->n;
  CK(cudaEventRecord(ctx->evc[0], ctx->stream));  // state buffers and flags (re)initialised
  const bool honours_a = prm->variant == SBG_GDSB;
  MultiStepArgs a;
  std::memset(&a, 0, sizeof a);
  a.n = int32_t(ctx->n);
  a.npad = int32_t(ctx->npad);
  a.R = int32_t(ctx->R);
  a.rpad = int32_t(ctx->rpad);
  a.k.a = honours_a ? float(prm->a) : 0.0f;
  a.k.c = float(prm->c);
  a.k.dt = float(prm->dt);
  a.M = prm->steps;
  a.t_begin = 0;
  a.nsteps = int32_t(prm->steps);
  a.a_rep = (honours_a && ctx->d_arep && ctx->arep_n == ctx->R) ? ctx->d_arep : nullptr;
  const int cur = ctx->g_cur;
  // Copies (second stream) are enqueued BEFORE the launch, which waits on nothing but the
  // flags: with pinned buffers the copies of later groups overlap the earlier groups' steps;
  // with pageable buffers, a serialising profiler or CUDA_LAUNCH_BLOCKING the copies simply
  // complete first (the kernel can never wait on work queued behind it).
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->evc[0], 0));
  for (int g = 0; g < nflags; ++g) {  // flag g covers replica rows [r0, r0 + rows)
    const int64_t r0 = g < rbg ? int64_t(g) * nr : int64_t(rbg) * nr * (g - rbg + 1);
    const int64_t rows = std::min<int64_t>(R - r0, g < rbg ? int64_t(nr) : int64_t(rbg) * nr);
    if (rows > 0) {
      CK(cudaMemcpy2DAsync(ctx->dX + r0 * ctx->npad, pitch, x0 + r0 * ctx->n, w, w, rows, cudaMemcpyHostToDevice,
                           ctx->cstream));
      CK(cudaMemcpy2DAsync(ctx->dY + r0 * ctx->npad, pitch, y0 + r0 * ctx->n, w, w, rows, cudaMemcpyHostToDevice,
                           ctx->cstream));
    }
    // stream-ordered flag write (with the default memory barrier: the rows are visible first)
    if (write_value(reinterpret_cast<CUstream>(ctx->cstream), reinterpret_cast<CUdeviceptr>(ctx->d_ready + g), 1u,
                    0) != CUDA_SUCCESS)
      return ctx->fail(SBG_ERR_CUDA, "cuStreamWriteValue32 failed");
  }
  CK(cudaEventRecord(ctx->ev[7], ctx->stream));
  CK(cudaEventRecord(ctx->ev[3], ctx->stream));
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  int gm = 1;
  rc = launch_resident_default(ctx, cur, a, groups, ctx->d_ready, &gm);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->evc[1], ctx->cstream));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->evc[1], 0));
  ctx->g_cur = cur ^ int(prm->steps & 1);
  ctx->g_mode = gm;
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  return run_tail(ctx, prm, x_final, spins, energy, best_index, timing, /*advanced=*/true);
}

int sbg_run(sbg_ctx* ctx, const sbg_params* prm, int64_t R, const float* x0, const float* y0, float* x_final,
            int8_t* spins, double* energy, int64_t* best_index, sbg_timing* timing) {
  CHECK_CTX(ctx);
  int rc = validate_params(ctx, prm);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (x0 && y0 && R >= 1 && use_resident(ctx, prm->variant) && !dev_knob("SBG_RUN_SERIAL")) {
    CK(cudaEventRecord(ctx->ev[2], ctx->stream));
    rc = ensure_state(ctx, R);  // resident_ok depends on the padded replica count
    if (rc) return rc;
    if (resident_ok(ctx)) return run_pipelined(ctx, prm, R, x0, y0, x_final, spins, energy, best_index, timing);
  }
  CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  rc = sbg_set_state(ctx, R, x0, y0, nullptr);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev[7], ctx->stream));
  return run_tail(ctx, prm, x_final, spins, energy, best_index, timing);
}

int sbg_run_best(sbg_ctx* ctx, const sbg_params* prm, int64_t R, const float* x0, const float* y0,
                 int8_t* best_spins, double* best_energy, int64_t* best_index, double* energies,
                 sbg_timing* timing) {
  CHECK_CTX(ctx);
  if (!best_spins || !best_energy || !best_index)
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "sbg_run_best needs best_spins, best_energy and best_index");
  ctx->tail_best_spins = best_spins;
  ctx->tail_best_energy = best_energy;
  const int rc = sbg_run(ctx, prm, R, x0, y0, nullptr, nullptr, energies, best_index, timing);
  ctx->tail_best_spins = nullptr;
  ctx->tail_best_energy = nullptr;
  return rc;
}

int sbg_run_seeded(sbg_ctx* ctx, const sbg_params* prm, int64_t R, int32_t init_mode, uint64_t master,
                   uint64_t tag, int64_t offset, int8_t* spins, double* energy, int64_t* best_index,
                   sbg_timing* timing) {
  CHECK_CTX(ctx);
  int rc = validate_params(ctx, prm);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  CK(cudaEventRecord(ctx->ev[2], ctx->stream));
  CK(cudaEventRecord(ctx->ev[7], ctx->stream));
  rc = sbg_init_state(ctx, R, init_mode, master, tag, offset);
  if (rc) return rc;
  return run_tail(ctx, prm, nullptr, spins, energy, best_index, timing);
}

// ------------------------------------------------------------------ row sharding (C5)

int sbg_gen_couplings_hash_pm1(sbg_ctx* ctx, int64_t n_global, int32_t world, int32_t rank, uint64_t seed) {
  CHECK_CTX(ctx);
  return gen_rows_common(ctx, n_global, world, rank, seed, GEN_HASH);
}

int sbg_gen_couplings_dense_pm1_rows(sbg_ctx* ctx, int64_t n_global, int32_t world, int32_t rank, uint64_t seed) {
  CHECK_CTX(ctx);
  return gen_rows_common(ctx, n_global, world, rank, seed, GEN_EXACT);
}

int sbg_get_couplings_i8(sbg_ctx* ctx, int64_t row_begin, int64_t rows, int8_t* J) {
  CHECK_CTX(ctx);
  if (ctx->kind != KIND_DENSE_I8) return ctx->fail(SBG_ERR_STATE, "int8 dense couplings not set");
  if (!J || row_begin < 0 || rows < 0 || row_begin + rows > ctx->n)
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad row range");
  if (rows == 0) return SBG_OK;
  CK(cudaSetDevice(ctx->device));
  const int64_t cols = ctx->sharded ? ctx->n_global : ctx->n;
  const int64_t ld = ctx->sharded ? ctx->kpad : ctx->npad;
  CK(cudaMemcpy2DAsync(J, cols, ctx->dJ + row_begin * ld, ld, cols, rows, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SBG_OK;
}

int sbg_set_couplings_rows_i8(sbg_ctx* ctx, int64_t n_global, int32_t world, int32_t rank, const int8_t* Jrows) {
  CHECK_CTX(ctx);
  if (n_global < 1 || world < 1 || world > 8 || rank < 0 || rank >= world || !Jrows)
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "bad row-shard arguments");
  const int64_t kpad = round_up(n_global, int64_t(256) * world);  // 256-row slabs: whole CTA pairs
  const int64_t rows = kpad / world;  // multiple of 128
  const int64_t row0 = int64_t(rank) * rows;
  const int64_t valid = std::max<int64_t>(0, std::min<int64_t>(rows, n_global - row0));
  for (int64_t i = 0; i < valid; ++i) {
    if (Jrows[i * n_global + row0 + i] != 0) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "coupling diagonal must be zero");
    for (int64_t j = 0; j < n_global; ++j)
      if (Jrows[i * n_global + j] == -128)
        return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "int8 couplings must lie in [-127, 127]");
  }
  CK(cudaSetDevice(ctx->device));
  cudaStreamSynchronize(ctx->stream);
  free_state(ctx);
  cudaFree(ctx->dJ);
  cudaFree(ctx->dJ4);
  ctx->dJ4 = nullptr;
  ctx->dJ = nullptr;
  CK(cudaMalloc(&ctx->dJ, size_t(rows) * kpad));
  CK(cudaMemsetAsync(ctx->dJ, 0, size_t(rows) * kpad, ctx->stream));
  if (valid > 0)
    CK(cudaMemcpy2DAsync(ctx->dJ, kpad, Jrows, n_global, n_global, valid, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->kind = KIND_DENSE_I8;
  ctx->energy_scale = 1.0;
  ctx->sharded = true;
  ctx->n = valid;
  ctx->npad = rows;
  ctx->n_global = n_global;
  ctx->kpad = kpad;
  ctx->row0 = row0;
  ctx->num_m_total = kpad / 128;
  ctx->done_base = 0;
  ctx->peer_g0.clear();
  ctx->peer_g1.clear();
  ctx->peer_done.clear();
  if (valid == 0) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "rank owns no spins (too many ranks for n)");
  const int rc = encode_2d_u8(ctx, &ctx->tmJ, ctx->dJ, kpad, rows, 128, 128);
  return rc ? rc : build_q4(ctx, rows, kpad);
}

int sbg_shard_info(const sbg_ctx* ctx, int64_t* row0, int64_t* rows_valid, int64_t* rows_padded, int64_t* kpad) {
  if (!ctx || !ctx->sharded) return SBG_ERR_STATE;
  if (row0) *row0 = ctx->row0;
  if (rows_valid) *rows_valid = ctx->n;
  if (rows_padded) *rows_padded = ctx->npad;
  if (kpad) *kpad = ctx->kpad;
  return SBG_OK;
}

int sbg_shard_buffers(sbg_ctx* ctx, void** g0, void** g1, void** done) {
  CHECK_CTX(ctx);
  if (!ctx->sharded || !ctx->dG[0]) return ctx->fail(SBG_ERR_STATE, "row shard with state required");
  if (g0) *g0 = ctx->dG[0];
  if (g1) *g1 = ctx->dG[1];
  if (done) *done = ctx->d_done;
  return SBG_OK;
}

int sbg_shard_set_peers(sbg_ctx* ctx, int32_t npeers, void* const* g0, void* const* g1, void* const* done) {
  CHECK_CTX(ctx);
  if (!ctx->sharded) return ctx->fail(SBG_ERR_STATE, "not a row shard");
  if (npeers < 0 || npeers > MAX_PEERS) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "at most 7 peers");
  ctx->peer_g0.assign(size_t(npeers), nullptr);
  ctx->peer_g1.assign(size_t(npeers), nullptr);
  ctx->peer_done.assign(size_t(npeers), nullptr);
  for (int i = 0; i < npeers; ++i) {
    ctx->peer_g0[size_t(i)] = static_cast<uint8_t*>(g0[i]);
    ctx->peer_g1[size_t(i)] = static_cast<uint8_t*>(g1[i]);
    ctx->peer_done[size_t(i)] = static_cast<uint32_t*>(done[i]);
  }
  CK(cudaSetDevice(ctx->device));
  if (!ctx->d_err) CK(cudaMalloc(&ctx->d_err, sizeof(uint32_t)));
  CK(cudaMemsetAsync(ctx->d_err, 0, sizeof(uint32_t), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_done, 0, sizeof(uint32_t) * (ctx->rpad / 16 + 1), ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->done_base = 0;
  return SBG_OK;
}

// Build this shard's slab of the step-0 B operand (sign variants) in the local G buffer.
int sbg_shard_prepare(sbg_ctx* ctx, int32_t variant) {
  CHECK_CTX(ctx);
  if (!ctx->sharded || !ctx->dX) return ctx->fail(SBG_ERR_STATE, "row shard with state required");
  if (!is_sign_variant(variant)) return ctx->fail(SBG_ERR_UNSUPPORTED, "row sharding supports dsb/gdsb");
  CK(cudaSetDevice(ctx->device));
  if (q4_stream(ctx)) {
    const size_t tot = size_t(ctx->rpad) * (ctx->npad / 2);
    prep_sign4_kernel<<<grid_for(ctx, tot, 256), 256, 0, ctx->stream>>>(
        ctx->dX, ctx->dG[ctx->g_cur], int32_t(ctx->n), int32_t(ctx->npad), int32_t(ctx->R), int32_t(ctx->rpad),
        ctx->kpad / 2, ctx->row0);
    CK(cudaGetLastError());
    ++ctx->launches;
    ctx->g_mode = 2;
  } else {
    int rc = prep_planes(ctx, ctx->dX, ctx->dG[ctx->g_cur], 1, ctx->R, ctx->rpad, /*into_global=*/true);
    if (rc) return rc;
    ctx->g_mode = 1;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return SBG_OK;
}

// Copy this shard's slab of the current B operand into every peer's buffer.
int sbg_shard_push_slab(sbg_ctx* ctx) {
  CHECK_CTX(ctx);
  if (!ctx->sharded) return ctx->fail(SBG_ERR_STATE, "not a row shard");
  CK(cudaSetDevice(ctx->device));
  for (size_t i = 0; i < ctx->peer_g0.size(); ++i) {
    const int64_t kb = ctx->g_mode == 2 ? 2 : 1;  // spins per byte (packed e2m1 plane)
    uint8_t* dst = (ctx->g_cur == 0 ? ctx->peer_g0[i] : ctx->peer_g1[i]) + ctx->row0 / kb;
    const uint8_t* src = ctx->dG[ctx->g_cur] + ctx->row0 / kb;
    CK(cudaMemcpy2DAsync(dst, ctx->kpad / kb, src, ctx->kpad / kb, ctx->npad / kb, ctx->R, cudaMemcpyDefault,
                         ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return SBG_OK;
}

// Test-only emulation of `nranks` row shards of ONE GPU as ONE cooperative launch of the e2m1
// CTA-pair kernel (FUSED): every rank keeps its own J rows, state, G buffers and done counter,
// wired to the others exactly as for separate GPUs (sbg_shard_set_peers), and runs m_begin ..
// m_end in one multi-step schedule on its own group of 2 * floor(sms / (2 nranks)) CTAs, so the
// cross-rank multi-step waits (system-scope acquire/release, slab pushes from the epilogue)
// execute as they would over NVLink. (Ranks that wait on one another must never be separate
// launches on one GPU: nothing guarantees they are co-resident.)
int sbg_shard_advance_fused(sbg_ctx* const* ctxs, int32_t nranks, const sbg_params* prm, uint64_t m_begin,
                            uint64_t m_end) {
  if (!ctxs || nranks < 2 || nranks > MAX_PEERS + 1) return SBG_ERR_INVALID_ARGUMENT;
  sbg_ctx* ctx = ctxs[0];
  CHECK_CTX(ctx);
  for (int r = 0; r < nranks; ++r) {
    sbg_ctx* c = ctxs[r];
    CHECK_CTX(c);
    int rc = validate_params(c, prm);
    if (rc) return rc;
    if (!c->sharded || !c->dX || c->R < 1) return ctx->fail(SBG_ERR_STATE, "rank %d: row shard with state required", r);
    if (c->device != ctx->device) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "fused ranks must share one device");
    if (!is_sign_variant(prm->variant) || !q4_stream(c) || c->g_mode != 2)
      return ctx->fail(SBG_ERR_UNSUPPORTED, "rank %d: fused emulation needs e2m1 shards after sbg_shard_prepare", r);
    if (int(c->peer_done.size()) != nranks - 1 || c->R != ctx->R || c->rpad != ctx->rpad || c->kpad != ctx->kpad ||
        c->npad != ctx->npad || c->g_cur != ctx->g_cur)
      return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "rank %d: shards must be wired to each other and alike", r);
  }
  if (m_end > prm->steps || m_begin > m_end)
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "state already at the final step");
  CK(cudaSetDevice(ctx->device));
  for (int r = 1; r < nranks; ++r) CK(cudaStreamSynchronize(ctxs[r]->stream));  // their prep is done
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  if (m_end == m_begin) {
    CK(cudaEventRecord(ctx->ev[1], ctx->stream));
    return SBG_OK;
  }
  const bool honours_a = prm->variant == SBG_GDSB;
  PhaseConsts k;
  k.a = honours_a ? float(prm->a) : 0.0f;
  k.c = float(prm->c);
  k.dt = float(prm->dt);
  k.inv = 0.0f;
  const int cur = ctx->g_cur;
  const int32_t ns = int32_t(m_end - m_begin);
  std::vector<MultiStepArgs> args(static_cast<size_t>(nranks));
  std::vector<TmaMaps> maps(static_cast<size_t>(nranks));
  for (int r = 0; r < nranks; ++r) {
    sbg_ctx* c = ctxs[r];
    MultiStepArgs& a = args[size_t(r)];
    std::memset(&a, 0, sizeof a);
    a.n = int32_t(c->n);
    a.npad = int32_t(c->npad);
    a.R = int32_t(c->R);
    a.rpad = int32_t(c->rpad);
    a.num_m = int32_t(c->npad / 128);
    a.num_n = int32_t(c->rpad / NPAIR_SIGN);
    a.k = k;
    a.M = prm->steps;
    a.t_begin = m_begin;
    a.nsteps = ns;
    a.done = c->d_done;
    a.kpad = int32_t(c->kpad);
    a.num_m_total = int32_t(c->num_m_total);
    a.col0 = int32_t(c->row0);
    a.done_base = c->done_base;
    a.g_ld = c->kpad / 2;
    a.npeers = int32_t(c->peer_done.size());
    a.err = c->d_err;
    for (int pr = 0; pr < a.npeers; ++pr) {
      a.peer_g[0][pr] = cur == 0 ? c->peer_g1[size_t(pr)] : c->peer_g0[size_t(pr)];
      a.peer_g[1][pr] = cur == 0 ? c->peer_g0[size_t(pr)] : c->peer_g1[size_t(pr)];
      a.peer_done[pr] = c->peer_done[size_t(pr)];
    }
    a.ksplit = 1;
    maps[size_t(r)] = c->pqmaps_sign[cur];
  }
  // rank tables in device memory (CUtensorMap needs 64-byte alignment: cudaMalloc gives 256)
  const size_t abytes = sizeof(MultiStepArgs) * size_t(nranks), mbytes = sizeof(TmaMaps) * size_t(nranks);
  const size_t moff = (mbytes + 255) / 256 * 256;
  if (ctx->fused_cap < moff + abytes) {
    cudaFree(ctx->d_fused);
    ctx->d_fused = nullptr;
    ctx->fused_cap = 0;
    CK(cudaMalloc(&ctx->d_fused, moff + abytes));
    ctx->fused_cap = moff + abytes;
  }
  uint8_t* dmaps = static_cast<uint8_t*>(ctx->d_fused);
  uint8_t* dargs = dmaps + moff;
  CK(cudaMemcpyAsync(dmaps, maps.data(), mbytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dargs, args.data(), abytes, cudaMemcpyHostToDevice, ctx->stream));
  MultiStepArgs a0 = args[0];
  a0.ranks = nranks;
  a0.rank_args = reinterpret_cast<const MultiStepArgs*>(dargs);
  a0.rank_maps = reinterpret_cast<const TmaMaps*>(dmaps);
  using Cfg = PairStepCfg<1, NPAIR_SIGN, 5, 2, 16, true>;
  auto kern = gsb_multistep_pair_kernel<1, NPAIR_SIGN, 5, 2, 16, true, 1, true>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
  const int cpr = 2 * ((ctx->sms / 2) / nranks);
  CK(launch_persistent(kern, cpr * nranks, Cfg::THREADS, Cfg::SMEM_BYTES, ctx->stream, maps[0], a0));
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // the other ranks' streams see the results
  for (int r = 0; r < nranks; ++r) {
    sbg_ctx* c = ctxs[r];
    ++c->launches;
    c->done_base += uint32_t(ns) * uint32_t(c->num_m_total);
    c->g_cur = cur ^ int(ns & 1);
    const int rc = shard_wait_check(c);
    if (rc) return ctx->fail(SBG_ERR_CUDA, "rank %d: %s", r, c->err.c_str());
  }
  return SBG_OK;
}

// Export this shard's buffers for cross-process peers (3 CUDA IPC handles, 64 B each).
int sbg_shard_ipc_export(sbg_ctx* ctx, void* out192) {
  CHECK_CTX(ctx);
  if (!ctx->sharded || !ctx->dG[0] || !out192) return ctx->fail(SBG_ERR_STATE, "row shard with state required");
  CK(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h[3];
  CK(cudaIpcGetMemHandle(&h[0], ctx->dG[0]));
  CK(cudaIpcGetMemHandle(&h[1], ctx->dG[1]));
  CK(cudaIpcGetMemHandle(&h[2], ctx->d_done));
  std::memcpy(out192, h, sizeof h);
  return SBG_OK;
}

int sbg_shard_ipc_open(sbg_ctx* ctx, const void* in192, void** g0, void** g1, void** done) {
  CHECK_CTX(ctx);
  if (!in192) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "null handles");
  CK(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h[3];
  std::memcpy(h, in192, sizeof h);
  void* p[3] = {nullptr, nullptr, nullptr};
  for (int i = 0; i < 3; ++i) CK(cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess));
  *g0 = p[0];
  *g1 = p[1];
  *done = p[2];
  return SBG_OK;
}

// This shard's share of E2 (sum over its spins i of s_i (J s)_i), from the full sign
// plane G[cur] (all spins, sign variants after a step or sbg_shard_prepare + push).
int sbg_readout_partial(sbg_ctx* ctx, int64_t* e2) {
  CHECK_CTX(ctx);
  if (!ctx->sharded || !ctx->dX || (ctx->g_mode != 1 && ctx->g_mode != 2))
    return ctx->fail(SBG_ERR_STATE, "sign-variant row shard required");
  CK(cudaSetDevice(ctx->device));
  const int8_t* plane = reinterpret_cast<const int8_t*>(ctx->dG[ctx->g_cur]);
  const CUtensorMap* pmap = &ctx->tmG_sign[ctx->g_cur];
  if (ctx->g_mode == 2) {
    // packed e2m1 signs of all spins -> a byte-per-spin plane in a private buffer. Not the other
    // G buffer: peers already on their next step push their slabs of G_{t+1} into it over
    // NVLink with no cross-rank sync against this readout.
    if (!ctx->dSignAll || ctx->sign_all_bytes != size_t(ctx->rpad) * ctx->kpad) {
      cudaFree(ctx->dSignAll);
      ctx->dSignAll = nullptr;
      ctx->sign_all_bytes = size_t(ctx->rpad) * ctx->kpad;
      CK(cudaMalloc(&ctx->dSignAll, ctx->sign_all_bytes));
      int rc = encode_2d_u8(ctx, &ctx->tmSignAll, ctx->dSignAll, ctx->kpad, ctx->rpad, 128, BN_SIGN);
      if (rc) return rc;
    }
    const size_t tot = size_t(ctx->rpad) * ctx->kpad;
    unpack_sign4_kernel<<<grid_for(ctx, tot, 256), 256, 0, ctx->stream>>>(ctx->dG[ctx->g_cur], ctx->dSignAll,
                                                                         ctx->kpad, int32_t(ctx->rpad));
    CK(cudaGetLastError());
    ++ctx->launches;
    plane = ctx->dSignAll;
    pmap = &ctx->tmSignAll;
  }
  CK(cudaMemsetAsync(ctx->dE2, 0, sizeof(unsigned long long) * ctx->rpad, ctx->stream));
  StepArgs a = base_args(ctx, BN_SIGN, ctx->R, ctx->rpad);
  a.sign_in = plane + ctx->row0;
  a.sign_ld = ctx->kpad;
  a.e2 = ctx->dE2;
  int rc = launch_step<1, BN_SIGN, EpiMode::Readout>(ctx, *pmap, a);
  if (rc) return rc;
  CK(cudaMemcpyAsync(e2, ctx->dE2, sizeof(long long) * ctx->R, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return shard_wait_check(ctx);
}

// Per-replica control strength A (a_rep[r] for replica r of the current state,
// R values): one launch then covers a whole A-sweep column (bench.cpp:143-197's
// run_sweep_cell fan-out over A). NULL clears it. Ignored by bsb/dsb (engine.cpp:64).
int sbg_set_replica_a(sbg_ctx* ctx, int64_t R, const float* a) {
  CHECK_CTX(ctx);
  CK(cudaSetDevice(ctx->device));
  if (!a) {
    ctx->arep_n = 0;
    return SBG_OK;
  }
  if (R < 1) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "replica count must be >= 1");
  for (int64_t r = 0; r < R; ++r)
    if (!(a[r] >= 0.0f)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "A must be >= 0");
  cudaFree(ctx->d_arep);
  ctx->d_arep = nullptr;
  CK(cudaMalloc(&ctx->d_arep, sizeof(float) * size_t(R)));
  CK(cudaMemcpy(ctx->d_arep, a, sizeof(float) * size_t(R), cudaMemcpyHostToDevice));
  ctx->arep_n = R;
  return SBG_OK;
}

int sbg_synchronize(sbg_ctx* ctx) {
  CHECK_CTX(ctx);
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  return shard_wait_check(ctx);
}

int sbg_state_device(sbg_ctx* ctx, float** x, float** y, float** p, int64_t* ld, int64_t* rpad) {
  CHECK_CTX(ctx);
  if (!ctx->dX) return ctx->fail(SBG_ERR_STATE, "no state");
  if (int rc = csr_sync(ctx)) return rc;
  if (x) *x = ctx->dX;
  if (y) *y = ctx->dY;
  if (p) *p = ctx->dP;
  if (ld) *ld = ctx->npad;
  if (rpad) *rpad = ctx->rpad;
  return SBG_OK;
}

int sbg_success_tts(int64_t hits, int64_t n_rep, double t_com, double* out) {
  // success_from_counts + time_to_solution, bench.cpp:15-26, :52-68
  if (!out) return SBG_ERR_INVALID_ARGUMENT;
  if (n_rep <= 0 || hits < 0 || hits > n_rep) return SBG_ERR_INVALID_ARGUMENT;
  const double p = double(hits) / double(n_rep);
  out[0] = p;
  out[1] = std::sqrt((p - p * p) / double(n_rep));
  if (!(t_com > 0.0) || !(p > 0.0)) return SBG_ERR_INVALID_ARGUMENT;
  if (p > 0.99) {
    out[2] = t_com;
    out[3] = 0.0;
  } else {
    const double log_miss = std::log1p(-p);
    out[2] = t_com * std::log(0.01) / log_miss;
    out[3] = out[2] * out[1] / ((1.0 - p) * std::fabs(log_miss));
  }
  return SBG_OK;
}

int sbg_tune_wigner_f64(int64_t n, const double* J, double d_t, double* c, double* dt) {
  // auto_tune(wigner): spectral.cpp:298-305 with offdiagonal_sigma (:254-266)
  if (n < 2 || !J || !c || !dt) return SBG_ERR_INVALID_ARGUMENT;
  if (!(d_t > 0.0)) return SBG_ERR_INVALID_ARGUMENT;
  double sum_sq = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j)
      if (j != i) sum_sq += J[i * n + j] * J[i * n + j];
  const double sigma = std::sqrt(sum_sq / (double(n) * double(n - 1)));
  if (sigma == 0.0) return SBG_ERR_INVALID_ARGUMENT;  // degenerate instance
  const double edge = 2.0 * std::sqrt(double(n)) * sigma;
  *c = 1.0 / edge;
  *dt = d_t * std::sqrt(2.0 / (1.0 - (-edge) / edge));
  return SBG_OK;
}

int sbg_extreme_eigenvalues(sbg_ctx* ctx, double tol, uint64_t max_iters, sbg_spectral* out, double* v_max,
                            double* v_min) {
  CHECK_CTX(ctx);
  if (!out) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "null output");
  *out = sbg_spectral{};
  JView jv;
  int rc = make_jview(ctx, &jv);
  if (rc) return rc;
  const int64_t n = jv.n;
  // extreme_eigenvalues argument checks, in order (spectral.cpp:209-213)
  if (n < 2) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "extreme_eigenvalues needs n >= 2");
  if (!(tol > 0.0)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "tolerance must be positive");
  CK(cudaSetDevice(ctx->device));
  double sum_sq = 0.0, beta = 0.0;
  if ((rc = row_stats(ctx, jv, &sum_sq, &beta))) return rc;
  if (beta == 0.0) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "degenerate instance: all couplings zero");
  if (max_iters == 0) max_iters = 10 * uint64_t(n);
  if (n <= 32) {  // closed form / Jacobi (spectral.cpp:215-216)
    double* d = nullptr;
    CK(cudaMalloc(&d, sizeof(double) * (2 + 2 * n)));
    spectral_small_kernel<<<1, 32, 0, ctx->stream>>>(jv, d);
    ++ctx->launches;
    std::vector<double> h(size_t(2 + 2 * n));
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d);
    if (e != cudaSuccess) return ctx->fail(SBG_ERR_CUDA, "small spectrum: %s", cudaGetErrorString(e));
    out->lambda_max = h[0];
    out->lambda_min = h[1];
    out->method = SBG_SPECTRAL_EXACT_SMALL;
    out->converged = 1;
    if (v_max) std::memcpy(v_max, &h[2], sizeof(double) * n);
    if (v_min) std::memcpy(v_min, &h[2 + n], sizeof(double) * n);
    return SBG_OK;
  }
  out->method = SBG_SPECTRAL_POWER_ITERATION;
  out->tolerance = tol;
  PowerOutcome hi, lo;
  if ((rc = power_end(ctx, jv, beta, +1.0, tol, max_iters, &hi, v_max))) return rc;
  out->lambda_max = hi.lambda;
  out->iterations = hi.iterations;
  if (!hi.converged) {
    out->lambda_min = std::nan("");
    return ctx->fail(SBG_ERR_CONVERGENCE, "lambda_max estimation did not converge in %s iterations (residual %s)",
                     std::to_string(max_iters).c_str(), std::to_string(hi.residual).c_str());
  }
  if ((rc = power_end(ctx, jv, beta, -1.0, tol, max_iters, &lo, v_min))) return rc;
  out->lambda_min = lo.lambda;
  out->iterations += lo.iterations;
  if (!lo.converged)
    return ctx->fail(SBG_ERR_CONVERGENCE, "lambda_min estimation did not converge in %s iterations (residual %s)",
                     std::to_string(max_iters).c_str(), std::to_string(lo.residual).c_str());
  out->converged = 1;
  return SBG_OK;
}

int sbg_auto_tune(sbg_ctx* ctx, int32_t mode, double d_t_factor, double tol, uint64_t max_iters, sbg_spectral* out) {
  CHECK_CTX(ctx);
  if (!out) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "null output");
  int rc;
  if (mode == SBG_TUNE_WIGNER) {  // spectral.cpp:298-305
    *out = sbg_spectral{};
    JView jv;
    if ((rc = make_jview(ctx, &jv))) return rc;
    CK(cudaSetDevice(ctx->device));
    const int64_t n = jv.n;
    double sum_sq = 0.0, beta = 0.0;
    if ((rc = row_stats(ctx, jv, &sum_sq, &beta))) return rc;
    const double sigma = n < 2 ? 0.0 : std::sqrt(sum_sq / (static_cast<double>(n) * static_cast<double>(n - 1)));
    if (sigma == 0.0) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "degenerate instance: all couplings zero");
    const double edge = 2.0 * std::sqrt(static_cast<double>(n)) * sigma;
    out->method = SBG_SPECTRAL_WIGNER;
    out->lambda_max = edge;
    out->lambda_min = -edge;
    out->converged = 1;
  } else if (mode == SBG_TUNE_NUMERICAL) {  // :306-320
    rc = sbg_extreme_eigenvalues(ctx, tol, max_iters, out, nullptr, nullptr);
    if (rc == SBG_ERR_CONVERGENCE) {
      if (!std::isfinite(out->lambda_max) || !std::isfinite(out->lambda_min) || !(out->lambda_max > 0.0) ||
          !(out->lambda_min < 0.0))
        return rc;
      out->converged = 0;  // tuned from the carried estimate (the reference warns on stderr)
    } else if (rc) {
      return rc;
    }
  } else {
    return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "unknown tune mode");
  }
  // tune_dt (spectral.cpp:277-286)
  if (!(out->lambda_max > 0.0)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "lambda_max must be positive");
  if (!(out->lambda_min < 0.0)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "lambda_min must be negative");
  if (!(d_t_factor > 0.0)) return ctx->fail(SBG_ERR_INVALID_ARGUMENT, "d_t_factor must be positive");
  out->d_t_factor = d_t_factor;
  out->c = 1.0 / out->lambda_max;
  out->dt = d_t_factor * std::sqrt(2.0 / (1.0 - out->lambda_min / out->lambda_max));
  return SBG_OK;
}

}  // extern "C"
