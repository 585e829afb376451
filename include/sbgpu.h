/* sbgpu — B200-native generalized simulated bifurcation (GSB), C ABI.
 *
 * This is the drop-in boundary for the reference's per-step hot path.
 * The reference (arxiv/paper_2508_17655, `sbopt`, /root/reference/proj/core)
 * exposes that path only as a C++ library with no FFI; each entry point below
 * names the reference interface it replaces (file:line relative to
 * /root/reference/proj/core). Plain pointers and sizes only; nothing throws
 * across this ABI: every call returns an SBG_* code and the message is kept in
 * sbg_last_error(ctx). The C++ wrapper include/sbgpu.hpp maps the codes back
 * to the reference's exception types (std::invalid_argument for argument
 * errors, engine.cpp:16-21/:57-60; std::runtime_error otherwise).
 *
 * Layouts: couplings J are dense row-major n x n (or CSR); replica states are
 * replica-major R x n (replica r's vector contiguous), fp32 on the device.
 * The caller owns all host arrays; no caller pointer is retained after a call.
 * A context is single-threaded and bound to one CUDA device.
 */
#ifndef SBGPU_H
#define SBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBG_ABI_VERSION 1

/* return codes */
#define SBG_OK 0
#define SBG_ERR_INVALID_ARGUMENT 1 /* maps to std::invalid_argument */
#define SBG_ERR_OUT_OF_MEMORY 2
#define SBG_ERR_CUDA 3
#define SBG_ERR_NCCL 4
#define SBG_ERR_STATE 5 /* call order: no couplings / no state yet */
#define SBG_ERR_UNSUPPORTED 6
#define SBG_ERR_CONVERGENCE 7 /* maps to sbopt::ConvergenceError (spectral.hpp:38-47) */

/* Variant (engine.hpp:26 `enum class Variant { bsb, dsb, gbsb }`, plus GdSB:
 * sign-discretised field with per-spin nonlinear control). */
#define SBG_BSB 0
#define SBG_DSB 1
#define SBG_GBSB 2
#define SBG_GDSB 3

/* Initial-state generators (device side, bit-exact with the oracle).
 * UNIFORM_RANDOM / CHAOS_PROBE: init_state, engine.cpp:25-39 (x ~ U(-1,1) or
 * +-0.1; y = 0; p = 1), rounded to fp32; replica r seeded
 * derive_seed(master, {tag, offset + r}) (rng.hpp:26-31; batch_best_of uses
 * tag 3, bench.cpp:80). SMALL_UNIFORM: the BASELINE configs' x, y ~ U(-0.1,0.1)
 * (x drawn first, then y, each 0.1*uniform_symmetric() rounded to fp32), p = 1. */
#define SBG_INIT_UNIFORM_RANDOM 0
#define SBG_INIT_CHAOS_PROBE 1
#define SBG_INIT_SMALL_UNIFORM 2

typedef struct sbg_ctx sbg_ctx;

/* SolverConfig (engine.hpp:29-38) after resolve_config (engine.cpp:48-53):
 * dt and c already resolved. steps = M. a = A (ignored for bsb/dsb, :64). */
typedef struct sbg_params {
  int32_t variant;
  int32_t reserved;
  uint64_t steps;
  double dt;
  double c;
  double a;
} sbg_params;

/* Device-measured phases of the last sbg_run* call (CUDA events). */
typedef struct sbg_timing {
  double h2d_ms;
  double init_ms;
  double steps_ms;
  double readout_ms;
  double d2h_ms;
  double total_ms;
  int64_t kernel_launches;
} sbg_timing;

int sbg_abi_version(void);
const char* sbg_strerror(int code);

/* Context on one CUDA device. Replaces the per-call ThreadPool/scratch of the
 * reference (parallel.hpp:18-50, engine.cpp:67-68). */
int sbg_create(int device, sbg_ctx** out);
void sbg_destroy(sbg_ctx* ctx);
const char* sbg_last_error(const sbg_ctx* ctx);
int sbg_device_sm_count(const sbg_ctx* ctx);
const char* sbg_device_name(const sbg_ctx* ctx);

/* Couplings. Replace IsingInstance (model.hpp:46-70; invariants model.cpp:54-68:
 * symmetric, zero diagonal). Dense integer J is kept as int8 on the device. */
int sbg_set_couplings_dense_i8(sbg_ctx* ctx, int64_t n, const int8_t* J);
/* fp64 J as IsingInstance stores it: integral entries in [-127, 127] take the int8
 * path, anything else the fixed-point real-J path below. */
int sbg_set_couplings_dense_f64(sbg_ctx* ctx, int64_t n, const double* J);
/* 1 if the dense couplings also hold a packed e2m1 (FP4) copy, made at upload when every
 * entry lies in {0, +-1, +-2, +-3, +-4, +-6} (all +-1 instances): the sign variants'
 * resident kernel then multiplies with tcgen05 kind::mxf4 (exact integer fields, twice
 * the int8 rate); else 0 (int8 operands). */
int sbg_couplings_e2m1(const sbg_ctx* ctx);
/* Real-valued couplings (e.g. Sherrington-Kirkpatrick, BASELINE configs[3]): J is
 * held as a 24-bit fixed-point image J_int = rint(J * 2^s) (s maximal with
 * |J_int| < 2^23) in three byte planes; fields are exact integer sums scaled once
 * (fp32-accurate), energies exact for J_int then scaled by 2^-s. n <= 11000.
 * sbg_set_couplings_dense_f64 routes non-integral J here. */
int sbg_set_couplings_dense_f32(sbg_ctx* ctx, int64_t n, const float* J);
/* The scale exponent s of the fixed-point coupling image (0 for integer J). */
int sbg_coupling_scale_exp(const sbg_ctx* ctx);
/* gen_random_dense (model.cpp:144-159) generated on the device into int8, in the
 * reference's exact draw order (xoshiro jump-ahead per row segment, bit-identical
 * to the serial walk) -- any n, including C5's n = 100000 (10 GB). */
int sbg_gen_couplings_dense_pm1(sbg_ctx* ctx, int64_t n, uint64_t seed);
/* CSR (both triangles, ascending columns), int8 values: the sparse view of
 * the same IsingInstance. */
int sbg_set_couplings_csr_i8(sbg_ctx* ctx, int64_t n, int64_t nnz, const int32_t* rowptr,
                             const int32_t* col, const int8_t* val);
/* MAX-CUT graph ingestion straight to CSR (no dense fp64): CutGraph edges
 * (model.hpp:72-95; 0-based endpoints, checks of model.cpp:91-103 in input order)
 * mapped by maxcut_to_ising (model.cpp:134-142, J_ij = J_ji = -w). Weights must lie
 * in [-127, 127]. *total_weight (optional) receives W, so cut = (W - E) / 2. */
int sbg_set_couplings_graph(sbg_ctx* ctx, int64_t n, int64_t m, const int64_t* i, const int64_t* j,
                            const int64_t* w, int64_t* total_weight);
/* IsingInstance::from_entries (model.cpp:70-86; the JSON instance document's
 * [i, j, J_ij] triples): integer entries in [-127, 127] go to CSR when sparse
 * (2m < n^2/16), anything else to the dense paths. */
int sbg_set_couplings_entries_f64(sbg_ctx* ctx, int64_t n, int64_t m, const int64_t* i, const int64_t* j,
                                  const double* value);
int64_t sbg_n(const sbg_ctx* ctx);

/* Replica states. Replace SolverState (engine.hpp:40-47) x R.
 * sbg_set_state: host x, y, p (p may be NULL -> 1), each R x n, step index m = 0.
 * Domain: |x| <= 1, as every reference init produces (engine.cpp:25-39) and the walls keep
 * (engine.cpp:93-99); the continuous variants' fixed-point field q = rint(x 2^30) as four
 * signed base-256 digits is exact for |x| < 1.99 and undefined beyond. */
int sbg_set_state(sbg_ctx* ctx, int64_t R, const float* x, const float* y, const float* p);
/* Device-side init_state (see SBG_INIT_*), replicas offset .. offset+R-1. */
int sbg_init_state(sbg_ctx* ctx, int64_t R, int32_t mode, uint64_t master, uint64_t tag,
                   int64_t replica_offset);
/* Same with an explicit seed per replica (e.g. the sweep's derive_seed(seed,
 * {sweep, mi, ai, r}), bench.cpp:159). */
int sbg_init_state_seeds(sbg_ctx* ctx, int64_t R, int32_t mode, const uint64_t* seeds);
int sbg_get_state(sbg_ctx* ctx, float* x, float* y, float* p);

/* step() (engine.cpp:55-110) for every replica, m = m_begin .. m_end-1 of an
 * M-step run (params->steps = M). Validation as validate()/step()
 * (engine.cpp:16-21, :57-60). Asynchronous; see sbg_synchronize. */
int sbg_advance(sbg_ctx* ctx, const sbg_params* params, uint64_t m_begin, uint64_t m_end);

/* Readout: signs_from_positions (model.cpp:161-165) + ising_energy
 * (model.cpp:112-123) per replica + batch_best_of's winner rule (bench.cpp:84-87,
 * min energy, ties to the lowest index). Any output may be NULL.
 * spins: R x n int8; energy: R doubles; best_index/best_energy: scalars. */
int sbg_readout(sbg_ctx* ctx, int8_t* spins, double* energy, int64_t* best_index, double* best_energy);

/* batch_best_of's result only (bench.cpp:70-92): the winner's spins (n int8),
 * its energy and index, plus (optional) all R energies. Copies n + 8R bytes
 * instead of the R x n spin matrix. */
int sbg_readout_best(sbg_ctx* ctx, int8_t* best_spins, double* best_energy, int64_t* best_index,
                     double* energies);

/* Teacher-forced fields for parity (coupling_matvec, kernels.hpp:33-46):
 * F = J * S for S (R x n, entries +-1) -> int32 R x n, bit-exact; and the
 * fixed-point field the continuous variants use for x (R x n fp32). */
int sbg_fields_sign(sbg_ctx* ctx, int64_t R, const int8_t* S, int32_t* F);
int sbg_fields_fixed(sbg_ctx* ctx, int64_t R, const float* x, float* F);

/* run() (engine.cpp:112-139) batched over R replicas from host initial states:
 * H2D, M steps, readout, D2H, all inside the call. Outputs may be NULL. */
int sbg_run(sbg_ctx* ctx, const sbg_params* params, int64_t R, const float* x0, const float* y0,
            float* x_final, int8_t* spins, double* energy, int64_t* best_index, sbg_timing* timing);
/* batch_best_of's result (bench.cpp:70-92) from host initial states: sbg_run, then only the
 * winner crosses to the host -- its n spins (best_spins), energy and index (ties to the
 * lowest replica) -- plus, if non-NULL, the R energies. */
int sbg_run_best(sbg_ctx* ctx, const sbg_params* params, int64_t R, const float* x0, const float* y0,
                 int8_t* best_spins, double* best_energy, int64_t* best_index, double* energies,
                 sbg_timing* timing);
/* Same with device-generated initial states (sbg_init_state). */
int sbg_run_seeded(sbg_ctx* ctx, const sbg_params* params, int64_t R, int32_t init_mode,
                   uint64_t master, uint64_t tag, int64_t replica_offset, int8_t* spins,
                   double* energy, int64_t* best_index, sbg_timing* timing);

/* ---- Row sharding (C5: N too large for one GPU) ----------------------------
 * Rank `rank` of `world` owns spins [row0, row0 + rows) with rows = kpad/world,
 * kpad = n_global rounded up to 256*world; Jrows is its rows of J (valid x n_global,
 * row-major). Its x, y, p cover its spins for every replica; the B operand G (signs
 * of ALL spins) is replicated: each step's epilogue writes this rank's slab into
 * its own G and, over NVLink, into every peer's G, then releases per-replica-block
 * completion counters on every rank (the row-chunked coupling_matvec of
 * kernels.hpp:33-46 spread over GPUs). Sign variants only (dsb/gdsb).
 * Order: set_couplings_rows -> set_state/init_state -> (exchange buffers) ->
 * shard_set_peers -> shard_prepare -> shard_push_slab on all ranks -> barrier -> advance. */
int sbg_set_couplings_rows_i8(sbg_ctx* ctx, int64_t n_global, int32_t world, int32_t rank, const int8_t* Jrows);
int sbg_shard_info(const sbg_ctx* ctx, int64_t* row0, int64_t* rows_valid, int64_t* rows_padded, int64_t* kpad);
int sbg_shard_buffers(sbg_ctx* ctx, void** g0, void** g1, void** done);
int sbg_shard_set_peers(sbg_ctx* ctx, int32_t npeers, void* const* g0, void* const* g1, void* const* done);
int sbg_shard_prepare(sbg_ctx* ctx, int32_t variant);
int sbg_shard_push_slab(sbg_ctx* ctx);
/* Test-only: nranks (2..8) row shards living on ONE GPU, wired to each other with
 * sbg_shard_set_peers and prepared (sbg_shard_prepare + sbg_shard_push_slab), advanced from
 * m_begin to m_end in ONE cooperative launch of the e2m1 CTA-pair kernel, each rank on its own
 * group of CTAs: the multi-step cross-rank waits of K7 run as over NVLink, without separate
 * launches that wait on one another on one GPU. Timing: sbg_last_advance_ms(ctxs[0]). */
int sbg_shard_advance_fused(sbg_ctx* const* ctxs, int32_t nranks, const sbg_params* prm, uint64_t m_begin,
                            uint64_t m_end);
/* Device-generated +-1 couplings for large-N throughput runs: J_ij = J_ji = sign from
 * splitmix64(seed ^ (min(i,j) * n + max(i,j))), zero diagonal (i.i.d. uniform +-1 like
 * gen_random_dense, NOT its draw order; parity tests use the exact order at small n).
 * world == 1: the whole matrix; world > 1: rank's rows as sbg_set_couplings_rows_i8. */
int sbg_gen_couplings_hash_pm1(sbg_ctx* ctx, int64_t n_global, int32_t world, int32_t rank, uint64_t seed);
/* Row shard (layout of sbg_set_couplings_rows_i8) of gen_random_dense(n_global, seed)
 * in the reference's exact draw order, generated on the device; world == 1 is
 * sbg_gen_couplings_dense_pm1. */
int sbg_gen_couplings_dense_pm1_rows(sbg_ctx* ctx, int64_t n_global, int32_t world, int32_t rank, uint64_t seed);
/* Copies rows [row_begin, row_begin + rows) of the context's int8 couplings back
 * (row-major, n columns; for a shard, local rows of its rows_valid x n_global). */
int sbg_get_couplings_i8(sbg_ctx* ctx, int64_t row_begin, int64_t rows, int8_t* J);
/* CUDA IPC export/open of (G0, G1, done) for peers in other processes (192 bytes). */
int sbg_shard_ipc_export(sbg_ctx* ctx, void* out192);
int sbg_shard_ipc_open(sbg_ctx* ctx, const void* in192, void** g0, void** g1, void** done);
/* This rank's share of E2 = sum_i s_i (J s)_i over its spins; sum over ranks, energy = -E2/2. */
int sbg_readout_partial(sbg_ctx* ctx, int64_t* e2);

/* Per-replica control strength A for gbsb/gdsb (R values, each >= 0; NULL clears):
 * a whole A sweep (bench.cpp:143-197, run_sweep_cell over the A axis) in one launch.
 * Applies while the state has exactly R replicas. */
int sbg_set_replica_a(sbg_ctx* ctx, int64_t R, const float* a);

int sbg_synchronize(sbg_ctx* ctx);
/* Kernel launches issued by this context since creation (bench evidence). */
int64_t sbg_kernel_launches(const sbg_ctx* ctx);
/* Raw device pointers of the resident state (fp32, leading dimension ld). */
int sbg_state_device(sbg_ctx* ctx, float** x, float** y, float** p, int64_t* ld, int64_t* rpad);
/* Device-time of the most recent sbg_advance, ms (CUDA events on the ctx stream). */
double sbg_last_advance_ms(const sbg_ctx* ctx);

/* Statistics, bench.cpp:15-68 (success_from_counts + time_to_solution).
 * out = {p_s, delta_p_s, tts, delta_tts}. INVALID_ARGUMENT as the reference throws. */
int sbg_success_tts(int64_t hits, int64_t n_rep, double t_com_s, double* out4);
/* auto_tune, Wigner branch (spectral.cpp:298-305, :254-266, :277-286) on dense
 * fp64 J: c = 1/(2 sqrt(n) sigma), dt = d_t * sqrt(2 / (1 - lmin/lmax)) = d_t. */
int sbg_tune_wigner_f64(int64_t n, const double* J, double d_t, double* c, double* dt);

/* SpectralEstimate + TuningResult (spectral.hpp:17-34). */
#define SBG_SPECTRAL_POWER_ITERATION 0
#define SBG_SPECTRAL_WIGNER 1
#define SBG_SPECTRAL_EXACT_SMALL 2
#define SBG_TUNE_WIGNER 0
#define SBG_TUNE_NUMERICAL 1
typedef struct sbg_spectral {
  double lambda_max;
  double lambda_min; /* NaN when lambda_max did not converge */
  double c;          /* sbg_auto_tune only: 1 / lambda_max */
  double dt;         /* sbg_auto_tune only: d_t * sqrt(2 / (1 - lambda_min / lambda_max)) */
  double d_t_factor;
  double tolerance;  /* power iteration: tol; 0 for wigner / exact_small */
  uint64_t iterations;
  int32_t method;    /* SBG_SPECTRAL_* */
  int32_t converged; /* 0: auto_tune fell back to the carried estimate (the reference's warning) */
} sbg_spectral;

/* extreme_eigenvalues (spectral.cpp:207-246) of the context's couplings on the
 * device (dense int8, CSR int8, or the fixed-point real-J image): n == 2 closed
 * form, n <= 32 cyclic Jacobi, else Gershgorin-shifted power iteration on each
 * end -- bitwise the reference's estimates for integer couplings. max_iters == 0
 * means 10 n. Non-convergence returns SBG_ERR_CONVERGENCE with the carried
 * estimate in *out (lambda_min NaN if lambda_max failed). v_max / v_min: optional
 * n doubles each (the unit eigenvector estimates). */
int sbg_extreme_eigenvalues(sbg_ctx* ctx, double tol, uint64_t max_iters, sbg_spectral* out, double* v_max,
                            double* v_min);
/* auto_tune (spectral.cpp:294-326) on the context's couplings: mode
 * SBG_TUNE_WIGNER (sigma from the device couplings) or SBG_TUNE_NUMERICAL
 * (sbg_extreme_eigenvalues, keeping a finite carried estimate on non-convergence
 * with converged = 0, as the reference does after its warning). */
int sbg_auto_tune(sbg_ctx* ctx, int32_t mode, double d_t_factor, double tol, uint64_t max_iters, sbg_spectral* out);

#ifdef __cplusplus
}
#endif
#endif /* SBGPU_H */
