/* TEST INFRASTRUCTURE ONLY — the CPU checker for the sbgpu hot path.
 *
 * A plain-C restatement of the reference algorithm (sbopt, /root/reference/proj/core)
 * for everything the reference cannot run as-is: GdSB, injected BASELINE initial
 * states, int8/CSR/SK instances at sizes the fp64 dense reference cannot hold,
 * and the fp32 "mirror" of the exact op order the CUDA epilogue uses.
 * Each function cites the reference lines it follows. Only tests/, the smoke
 * check and bench.py's cpu_baseline/reference leg may load this library, and
 * only as the checker. It is pinned against the compiled reference
 * (oracle/_ref, see oracle/Makefile) by tests/test_oracle.py and the
 * committed golden vectors in tests/golden/.
 */
#ifndef SBG_ORACLE_H
#define SBG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Variant codes: 0 bsb, 1 dsb, 2 gbsb, 3 gdsb (engine.hpp:26 plus GdSB). */

/* ---- rng.hpp:17-77 ---------------------------------------------------- */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_derive_seed(uint64_t master, const uint64_t* keys, int nkeys);
void orc_xoshiro_next_n(uint64_t seed, int64_t count, uint64_t* out);

/* ---- instances -------------------------------------------------------- */
/* gen_random_dense (model.cpp:144-159) draw order, written as int8. */
void orc_gen_dense_i8(int64_t n, uint64_t seed, int8_t* J);
/* Rows [row0, row0+rows) of the same matrix, for instances too big to hold
 * whole (C5). Cost is O(row0*n) skipped draws. */
void orc_gen_dense_i8_rows(int64_t n, uint64_t seed, int64_t row0, int64_t rows, int8_t* Jrows);
/* Counter-based +-1 rows of sbg_gen_couplings_hash_pm1 (large-N throughput instance). */
void orc_gen_hash_pm1_rows(int64_t n, uint64_t seed, int64_t row0, int64_t rows, int8_t* Jrows);
/* Erdos-Renyi G(n, m) MAX-CUT graph (new; the reference has none): one
 * Xoshiro256pp(seed) stream, (i, j) = (next() % n, next() % n), self-loops and
 * duplicates rejected, then one random_sign() weight per accepted edge. */
int64_t orc_gen_er_edges(int64_t n, int64_t m, uint64_t seed, int32_t* ei, int32_t* ej, int8_t* w);
/* maxcut_to_ising (model.cpp:134-142): J = -w on both triangles, as CSR with
 * ascending columns. rowptr n+1, col/val 2m. */
void orc_edges_to_csr(int64_t n, int64_t m, const int32_t* ei, const int32_t* ej, const int8_t* w,
                      int32_t* rowptr, int32_t* col, int8_t* val);
/* Sherrington-Kirkpatrick J_ij ~ N(0, 1/n) fp32 (new): upper triangle row-major
 * from one Xoshiro256pp(seed), Box-Muller on uniform01 pairs, mirrored, zero diag. */
void orc_gen_sk_f32(int64_t n, uint64_t seed, float* J);

/* ---- initial states (layout [R][ld], replica-major) ------------------- */
/* BASELINE init: replica r uses Xoshiro256pp(derive_seed(master,{tag,r}));
 * x_i = (float)(0.1*uniform_symmetric()) for i<n, then y_i likewise; p = 1. */
void orc_init_small_uniform(int64_t n, int64_t ld, int64_t r0, int64_t R, uint64_t master,
                            uint64_t tag, float* x, float* y, float* p);
/* init_state (engine.cpp:25-39) rounded to fp32: x ~ U(-1,1) (or +-0.1 for
 * chaos_probe), y = 0, p = 1; seed derive_seed(master,{tag,r}) as batch_best_of
 * (bench.cpp:80) does with tag = 3. */
void orc_init_reference(int64_t n, int64_t ld, int64_t r0, int64_t R, uint64_t master, uint64_t tag,
                        int chaos_probe, float* x, float* y, float* p);

void orc_init_reference_seeds(int64_t n, int64_t ld, int64_t R, const uint64_t* seeds, int chaos_probe, float* x,
                              float* y, float* p);

/* ---- fp64 restatement of the reference step --------------------------- */
/* row_dot / coupling_matvec (kernels.hpp:14-46): 8 lanes, tail in lane 0. */
void orc_matvec_lanes_f64(int64_t n, const double* J, const double* v, double* out);
/* CSR equivalent of the same lane order. */
void orc_csr_matvec_lanes_f64(int64_t n, const int32_t* rowptr, const int32_t* col,
                              const double* val, const double* v, double* out);
/* step (engine.cpp:55-110) with GdSB added: a honoured for gbsb AND gdsb,
 * sign field for dsb AND gdsb. */
void orc_step_f64(int variant, int64_t n, const double* J, double* x, double* y, double* p,
                  uint64_t m, uint64_t M, double dt, double c, double a);

/* ---- fp32 mirror of the CUDA op order (bitwise reference for the GPU) --- */
/* Teacher-forced integer field F = J * S, S in {-1,+1}, layout [R][ld]. */
void orc_fields_i8(int64_t n, const int8_t* J, int64_t R, int64_t ld, const int8_t* S, int32_t* F);
/* Field the GPU uses for continuous x: F = fl32(sum_j J_ij q_j) * 2^-30 with
 * q_j = rint(x_j * 2^30) and the integer sum exact. */
void orc_fields_fixed_i8(int64_t n, const int8_t* J, int64_t R, int64_t ld, const float* x, float* F);
/* One step of all R replicas, dense int8 J. */
void orc_step_f32(int variant, int64_t n, const int8_t* J, int64_t R, int64_t ld, float* x, float* y,
                  float* p, uint64_t m, uint64_t M, float dt, float c, float a);
/* Same with a CSR int8 J (fields identical to the dense form on the dense view). */
void orc_step_f32_csr(int variant, int64_t n, const int32_t* rowptr, const int32_t* col,
                      const int8_t* val, int64_t R, int64_t ld, float* x, float* y, float* p,
                      uint64_t m, uint64_t M, float dt, float c, float a);
/* The elementwise phase alone (engine.cpp:86-103 in fp32, GPU op order). */
void orc_phase_f32(float F, float* x, float* y, float* p, float a, float c, float dt, float inv);

void orc_phase_batch_f32(int64_t count, const float* F, float* x, float* y, float* p, float a, float c, float dt,
                         uint64_t m, uint64_t M);

/* ---- readout ---------------------------------------------------------- */
/* E2[r] = sum_i s_i (J s)_i with s = sgn(x) (sgn(0)=+1, model.cpp:161-165);
 * energy = -E2/2 (model.cpp:112-123), exact for integer J. */
void orc_energy2_i8(int64_t n, const int8_t* J, int64_t R, int64_t ld, const float* x, int64_t* E2);
void orc_energy2_csr(int64_t n, const int32_t* rowptr, const int32_t* col, const int8_t* val,
                     int64_t R, int64_t ld, const float* x, int64_t* E2);
/* batch_best_of winner rule (bench.cpp:84-87): min, ties to lowest index. */
int64_t orc_argmin_i64(int64_t R, const int64_t* v);

/* ---- real-valued J (fixed-point image, GPU op order) ------------------- */
/* Quantise J like sbg_set_couplings_dense_f32; returns the scale exponent s. */
int orc_fx_quantize(int64_t n, const float* J, uint8_t* planes /* [3][n][n] */);
/* The fixed-point field alone (continuous variants: the 9 plane products of weight >= 2^16). */
void orc_fields_fx(int variant, int64_t n, const uint8_t* planes, int shift, int64_t R, int64_t ld, const float* x,
                   float* F);
void orc_step_f32_fx(int variant, int64_t n, const uint8_t* planes, int shift, int64_t R, int64_t ld, float* x,
                     float* y, float* p, uint64_t m, uint64_t M, float dt, float c, float a);
void orc_energy2_fx(int64_t n, const uint8_t* planes, int64_t R, int64_t ld, const float* x, int64_t* E2);

/* ---- statistics (bench.cpp:15-68) ------------------------------------- */
int orc_success_tts(int64_t hits, int64_t n_rep, double t_com, double* p_s, double* dp_s,
                    double* tts, double* dtts);

#ifdef __cplusplus
}
#endif
#endif
