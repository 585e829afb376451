/* TEST INFRASTRUCTURE ONLY — see sbg_oracle.h. Compile with -ffp-contract=off
 * (oracle/Makefile) so every fp operation below rounds exactly as written.
 * Citations are relative to /root/reference/proj/core/. */
#include "sbg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */

uint64_t orc_mix64(uint64_t z) { /* rng.hpp:17-21 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t orc_derive_seed(uint64_t master, const uint64_t* keys, int nkeys) { /* rng.hpp:26-31 */
  uint64_t h = orc_mix64(master + 0x9E3779B97F4A7C15ULL);
  for (int k = 0; k < nkeys; ++k) h = orc_mix64(h ^ (keys[k] + 0x9E3779B97F4A7C15ULL));
  return h;
}

typedef struct {
  uint64_t s[4];
} xo_t;

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static void xo_seed(xo_t* g, uint64_t seed) { /* rng.hpp:46-52 */
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) {
    z += 0x9E3779B97F4A7C15ULL;
    g->s[i] = orc_mix64(z);
  }
}

static inline uint64_t xo_next(xo_t* g) { /* rng.hpp:54-64 */
  uint64_t* s = g->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

static inline double xo_uniform01(xo_t* g) { /* rng.hpp:67 */
  return (double)(xo_next(g) >> 11) * 0x1.0p-53;
}
static inline double xo_uniform_symmetric(xo_t* g) { return 2.0 * xo_uniform01(g) - 1.0; } /* :70 */
static inline double xo_random_sign(xo_t* g) { return (xo_next(g) >> 63) ? -1.0 : 1.0; }  /* :73 */

void orc_xoshiro_next_n(uint64_t seed, int64_t count, uint64_t* out) {
  xo_t g;
  xo_seed(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = xo_next(&g);
}

/* ---------------------------------------------------------- instances */

void orc_gen_dense_i8(int64_t n, uint64_t seed, int8_t* J) { /* model.cpp:144-159 */
  xo_t g;
  xo_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) J[i * n + i] = 0;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = i + 1; j < n; ++j) {
      const int8_t v = (int8_t)xo_random_sign(&g);
      J[i * n + j] = v;
      J[j * n + i] = v;
    }
  }
}

void orc_gen_dense_i8_rows(int64_t n, uint64_t seed, int64_t row0, int64_t rows, int8_t* Jr) {
  /* Entry (i, j), i < j, is draw number i*n - i*(i+1)/2 + (j - i - 1) of the
   * stream. Row r needs its upper part (draws of row r) and its lower part
   * J[r][j] = J[j][r] for j < r (draws of earlier rows). Walk the stream once
   * up to the last needed draw. */
  xo_t g;
  xo_seed(&g, seed);
  const int64_t rend = row0 + rows;
  for (int64_t k = 0; k < rows; ++k) Jr[k * n + row0 + k] = 0;
  for (int64_t i = 0; i < n && i < rend; ++i) {
    for (int64_t j = i + 1; j < n; ++j) {
      const int8_t v = (int8_t)xo_random_sign(&g);
      if (i >= row0) Jr[(i - row0) * n + j] = v;
      if (j >= row0 && j < rend) Jr[(j - row0) * n + i] = v;
    }
  }
}

typedef struct {
  uint64_t* keys;
  int64_t cap;
} hset_t;

static int hset_insert(hset_t* h, uint64_t key) { /* 1 if inserted, 0 if present */
  uint64_t k1 = key + 1; /* 0 marks empty */
  uint64_t pos = orc_mix64(k1) & (uint64_t)(h->cap - 1);
  for (;;) {
    if (h->keys[pos] == 0) {
      h->keys[pos] = k1;
      return 1;
    }
    if (h->keys[pos] == k1) return 0;
    pos = (pos + 1) & (uint64_t)(h->cap - 1);
  }
}

int64_t orc_gen_er_edges(int64_t n, int64_t m, uint64_t seed, int32_t* ei, int32_t* ej, int8_t* w) {
  if (n < 2 || m > n * (n - 1) / 2) return -1;
  xo_t g;
  xo_seed(&g, seed);
  hset_t h;
  h.cap = 1;
  while (h.cap < 4 * m + 16) h.cap <<= 1;
  h.keys = (uint64_t*)calloc((size_t)h.cap, sizeof(uint64_t));
  int64_t got = 0;
  while (got < m) {
    const int64_t i = (int64_t)(xo_next(&g) % (uint64_t)n);
    const int64_t j = (int64_t)(xo_next(&g) % (uint64_t)n);
    if (i == j) continue;
    const uint64_t lo = (uint64_t)(i < j ? i : j), hi = (uint64_t)(i < j ? j : i);
    if (!hset_insert(&h, (hi << 32) | lo)) continue; /* same key as model.cpp:21-25 */
    ei[got] = (int32_t)i;
    ej[got] = (int32_t)j;
    ++got;
  }
  for (int64_t e = 0; e < m; ++e) w[e] = (int8_t)xo_random_sign(&g);
  free(h.keys);
  return m;
}

void orc_edges_to_csr(int64_t n, int64_t m, const int32_t* ei, const int32_t* ej, const int8_t* w,
                      int32_t* rowptr, int32_t* col, int8_t* val) {
  int32_t* deg = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  for (int64_t e = 0; e < m; ++e) {
    deg[ei[e]]++;
    deg[ej[e]]++;
  }
  rowptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) rowptr[i + 1] = rowptr[i] + deg[i];
  int32_t* fill = (int32_t*)calloc((size_t)n, sizeof(int32_t));
  for (int64_t e = 0; e < m; ++e) {
    const int32_t a = ei[e], b = ej[e];
    const int8_t v = (int8_t)(-w[e]); /* maxcut_to_ising: J = -w */
    col[rowptr[a] + fill[a]] = b;
    val[rowptr[a] + fill[a]++] = v;
    col[rowptr[b] + fill[b]] = a;
    val[rowptr[b] + fill[b]++] = v;
  }
  /* ascending columns inside each row (insertion sort; rows are short) */
  for (int64_t i = 0; i < n; ++i) {
    for (int32_t k = rowptr[i] + 1; k < rowptr[i + 1]; ++k) {
      const int32_t c = col[k];
      const int8_t v = val[k];
      int32_t t = k - 1;
      while (t >= rowptr[i] && col[t] > c) {
        col[t + 1] = col[t];
        val[t + 1] = val[t];
        --t;
      }
      col[t + 1] = c;
      val[t + 1] = v;
    }
  }
  free(deg);
  free(fill);
}

void orc_gen_sk_f32(int64_t n, uint64_t seed, float* J) {
  xo_t g;
  xo_seed(&g, seed);
  const double inv_sqrt_n = 1.0 / sqrt((double)n);
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < n; ++i) J[i * n + i] = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = i + 1; j < n; ++j) {
      const double u1 = xo_uniform01(&g);
      const double u2 = xo_uniform01(&g);
      const double z = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
      const float v = (float)(z * inv_sqrt_n);
      J[i * n + j] = v;
      J[j * n + i] = v;
    }
  }
}

/* ------------------------------------------------------- initial states */

void orc_init_small_uniform(int64_t n, int64_t ld, int64_t r0, int64_t R, uint64_t master,
                            uint64_t tag, float* x, float* y, float* p) {
  for (int64_t r = 0; r < R; ++r) {
    const uint64_t keys[2] = {tag, (uint64_t)(r0 + r)};
    xo_t g;
    xo_seed(&g, orc_derive_seed(master, keys, 2));
    for (int64_t i = 0; i < n; ++i) x[r * ld + i] = (float)(0.1 * xo_uniform_symmetric(&g));
    for (int64_t i = 0; i < n; ++i) y[r * ld + i] = (float)(0.1 * xo_uniform_symmetric(&g));
    for (int64_t i = 0; i < n; ++i) p[r * ld + i] = 1.0f;
    for (int64_t i = n; i < ld; ++i) x[r * ld + i] = y[r * ld + i] = p[r * ld + i] = 0.0f;
  }
}

void orc_init_reference(int64_t n, int64_t ld, int64_t r0, int64_t R, uint64_t master, uint64_t tag,
                        int chaos_probe, float* x, float* y, float* p) {
  for (int64_t r = 0; r < R; ++r) { /* engine.cpp:25-39 */
    const uint64_t keys[2] = {tag, (uint64_t)(r0 + r)};
    xo_t g;
    xo_seed(&g, orc_derive_seed(master, keys, 2));
    for (int64_t i = 0; i < n; ++i)
      x[r * ld + i] = chaos_probe ? (float)(0.1 * xo_random_sign(&g)) : (float)xo_uniform_symmetric(&g);
    for (int64_t i = 0; i < n; ++i) {
      y[r * ld + i] = 0.0f;
      p[r * ld + i] = 1.0f;
    }
    for (int64_t i = n; i < ld; ++i) x[r * ld + i] = y[r * ld + i] = p[r * ld + i] = 0.0f;
  }
}

/* ------------------------------------------------------- fp64 restatement */

static double row_dot(const double* a, const double* b, int64_t n) { /* kernels.hpp:14-30 */
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  double acc4 = 0.0, acc5 = 0.0, acc6 = 0.0, acc7 = 0.0;
  int64_t j = 0;
  for (; j + 8 <= n; j += 8) {
    acc0 += a[j + 0] * b[j + 0];
    acc1 += a[j + 1] * b[j + 1];
    acc2 += a[j + 2] * b[j + 2];
    acc3 += a[j + 3] * b[j + 3];
    acc4 += a[j + 4] * b[j + 4];
    acc5 += a[j + 5] * b[j + 5];
    acc6 += a[j + 6] * b[j + 6];
    acc7 += a[j + 7] * b[j + 7];
  }
  for (; j < n; ++j) acc0 += a[j] * b[j];
  return ((acc0 + acc1) + (acc2 + acc3)) + ((acc4 + acc5) + (acc6 + acc7));
}

void orc_matvec_lanes_f64(int64_t n, const double* J, const double* v, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = row_dot(J + i * n, v, n); /* kernels.hpp:33-46 */
}

void orc_csr_matvec_lanes_f64(int64_t n, const int32_t* rowptr, const int32_t* col,
                              const double* val, const double* v, double* out) {
  const int64_t full = 8 * (n / 8);
  for (int64_t i = 0; i < n; ++i) {
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int64_t j = col[k];
      acc[j < full ? (j & 7) : 0] += val[k] * v[j];
    }
    out[i] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  }
}

static int is_sign_variant(int v) { return v == 1 || v == 3; }
static int honours_a(int v) { return v == 2 || v == 3; }

void orc_step_f64(int variant, int64_t n, const double* J, double* x, double* y, double* p,
                  uint64_t m, uint64_t M, double dt, double c, double a_cfg) {
  /* engine.cpp:55-110; line 64 extended so GdSB keeps a. */
  const double a = honours_a(variant) ? a_cfg : 0.0;
  const double denom = (double)(M - m);
  double* g = (double*)malloc(sizeof(double) * (size_t)n);
  double* jx = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) g[i] = is_sign_variant(variant) ? (x[i] >= 0.0 ? 1.0 : -1.0) : x[i];
  orc_matvec_lanes_f64(n, J, g, jx);
  for (int64_t i = 0; i < n; ++i) { /* engine.cpp:86-103 */
    const double xi = x[i];
    const double pi = p[i] - (1.0 - a * xi * xi) * p[i] / denom;
    p[i] = pi;
    double yi = y[i] - (pi * xi - c * jx[i]) * dt;
    double xn = xi + yi * dt;
    if (xn > 1.0) {
      xn = 1.0;
      yi = 0.0;
    } else if (xn < -1.0) {
      xn = -1.0;
      yi = 0.0;
    }
    x[i] = xn;
    y[i] = yi;
  }
  free(g);
  free(jx);
}

/* ------------------------------------------------------- fp32 GPU mirror */

void orc_phase_f32(float F, float* xp, float* yp, float* pp, float a, float c, float dt, float inv) {
  /* engine.cpp:86-103 in the exact fp32 op order of the CUDA epilogue
   * (paper_2508_17655_b200/csrc/gsb_phase.cuh). No contraction. */
  const float x = *xp, y = *yp, p = *pp;
  const float ax2 = (a * x) * x;
  const float gmul = 1.0f - ax2;
  const float pn = p - (gmul * p) * inv; /* inv = RN(1/(M-m)), see step_f32_impl */
  const float t = pn * x - c * F;
  float yn = y - t * dt;
  float xn = x + yn * dt;
  if (xn > 1.0f) {
    xn = 1.0f;
    yn = 0.0f;
  } else if (xn < -1.0f) {
    xn = -1.0f;
    yn = 0.0f;
  }
  *xp = xn;
  *yp = yn;
  *pp = pn;
}

void orc_fields_i8(int64_t n, const int8_t* J, int64_t R, int64_t ld, const int8_t* S, int32_t* F) {
  for (int64_t r = 0; r < R; ++r) {
    const int8_t* s = S + r * ld;
    for (int64_t i = 0; i < n; ++i) {
      const int8_t* row = J + i * n;
      int32_t acc = 0;
      for (int64_t j = 0; j < n; ++j) acc += (int32_t)row[j] * (int32_t)s[j];
      F[r * ld + i] = acc;
    }
  }
}

static inline int32_t quant30(float x) { return (int32_t)lrintf(x * 0x1p30f); }

void orc_fields_fixed_i8(int64_t n, const int8_t* J, int64_t R, int64_t ld, const float* x, float* F) {
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t r = 0; r < R; ++r) {
    for (int64_t j = 0; j < n; ++j) q[j] = quant30(x[r * ld + j]);
    for (int64_t i = 0; i < n; ++i) {
      const int8_t* row = J + i * n;
      int64_t acc = 0;
      for (int64_t j = 0; j < n; ++j) acc += (int64_t)row[j] * (int64_t)q[j];
      F[r * ld + i] = (float)acc * 0x1p-30f;
    }
  }
  free(q);
}

static void fields_for(int variant, int64_t n, const int8_t* J, const int32_t* rowptr,
                       const int32_t* col, const int8_t* val, const float* xr, float* F,
                       int8_t* s, int32_t* q) {
  if (is_sign_variant(variant)) {
    for (int64_t j = 0; j < n; ++j) s[j] = xr[j] >= 0.0f ? 1 : -1;
  } else {
    for (int64_t j = 0; j < n; ++j) q[j] = quant30(xr[j]);
  }
  for (int64_t i = 0; i < n; ++i) {
    int64_t acc = 0;
    if (J) {
      const int8_t* row = J + i * n;
      if (is_sign_variant(variant))
        for (int64_t j = 0; j < n; ++j) acc += (int64_t)row[j] * s[j];
      else
        for (int64_t j = 0; j < n; ++j) acc += (int64_t)row[j] * q[j];
    } else {
      for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
        acc += (int64_t)val[k] * (is_sign_variant(variant) ? (int64_t)s[col[k]] : (int64_t)q[col[k]]);
    }
    F[i] = is_sign_variant(variant) ? (float)acc : (float)acc * 0x1p-30f;
  }
}

static void step_f32_impl(int variant, int64_t n, const int8_t* J, const int32_t* rowptr,
                          const int32_t* col, const int8_t* val, int64_t R, int64_t ld, float* x,
                          float* y, float* p, uint64_t m, uint64_t M, float dt, float c, float a_cfg) {
  const float a = honours_a(variant) ? a_cfg : 0.0f;
  const float inv = 1.0f / (float)(M - m); /* correctly rounded, == __frcp_rn on the GPU */
  float* F = (float*)malloc(sizeof(float) * (size_t)n);
  int8_t* s = (int8_t*)malloc((size_t)n);
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t r = 0; r < R; ++r) {
    float* xr = x + r * ld;
    fields_for(variant, n, J, rowptr, col, val, xr, F, s, q);
    for (int64_t i = 0; i < n; ++i) orc_phase_f32(F[i], xr + i, y + r * ld + i, p + r * ld + i, a, c, dt, inv);
  }
  free(F);
  free(s);
  free(q);
}

void orc_step_f32(int variant, int64_t n, const int8_t* J, int64_t R, int64_t ld, float* x, float* y,
                  float* p, uint64_t m, uint64_t M, float dt, float c, float a) {
  step_f32_impl(variant, n, J, NULL, NULL, NULL, R, ld, x, y, p, m, M, dt, c, a);
}

void orc_step_f32_csr(int variant, int64_t n, const int32_t* rowptr, const int32_t* col,
                      const int8_t* val, int64_t R, int64_t ld, float* x, float* y, float* p,
                      uint64_t m, uint64_t M, float dt, float c, float a) {
  step_f32_impl(variant, n, NULL, rowptr, col, val, R, ld, x, y, p, m, M, dt, c, a);
}

/* ---------------------------------------------------------------- readout */

void orc_energy2_i8(int64_t n, const int8_t* J, int64_t R, int64_t ld, const float* x, int64_t* E2) {
  int8_t* s = (int8_t*)malloc((size_t)n);
  for (int64_t r = 0; r < R; ++r) {
    for (int64_t j = 0; j < n; ++j) s[j] = x[r * ld + j] >= 0.0f ? 1 : -1; /* model.cpp:161-165 */
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) { /* model.cpp:112-123 */
      const int8_t* row = J + i * n;
      int64_t field = 0;
      for (int64_t j = 0; j < n; ++j) field += (int64_t)row[j] * s[j];
      total += field * s[i];
    }
    E2[r] = total;
  }
  free(s);
}

void orc_energy2_csr(int64_t n, const int32_t* rowptr, const int32_t* col, const int8_t* val,
                     int64_t R, int64_t ld, const float* x, int64_t* E2) {
  int8_t* s = (int8_t*)malloc((size_t)n);
  for (int64_t r = 0; r < R; ++r) {
    for (int64_t j = 0; j < n; ++j) s[j] = x[r * ld + j] >= 0.0f ? 1 : -1;
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) {
      int64_t field = 0;
      for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) field += (int64_t)val[k] * s[col[k]];
      total += field * s[i];
    }
    E2[r] = total;
  }
  free(s);
}

int64_t orc_argmin_i64(int64_t R, const int64_t* v) { /* bench.cpp:84-87 */
  int64_t best = 0;
  for (int64_t r = 1; r < R; ++r)
    if (v[r] < v[best]) best = r;
  return best;
}

/* ------------------------------------------------------------- statistics */

int orc_success_tts(int64_t hits, int64_t n_rep, double t_com, double* p_s, double* dp_s,
                    double* tts, double* dtts) {
  if (n_rep <= 0 || hits < 0 || hits > n_rep) return 1; /* bench.cpp:16-17 */
  const double p = (double)hits / (double)n_rep;
  *p_s = p;
  *dp_s = sqrt((p - p * p) / (double)n_rep);
  if (!(t_com > 0.0) || !(p > 0.0)) return 2; /* bench.cpp:53-54 */
  if (p > 0.99) {
    *tts = t_com;
    *dtts = 0.0;
  } else {
    const double log_miss = log1p(-p);
    *tts = t_com * log(0.01) / log_miss;
    *dtts = *tts * *dp_s / ((1.0 - p) * fabs(log_miss));
  }
  return 0;
}

/* ------------------------------------------- real-valued J, fixed-point mirror */

int orc_fx_quantize(int64_t n, const float* J, uint8_t* planes /* [3][n][n] */) {
  /* Host quantisation of sbg_set_couplings_dense_f32 (csrc/sbgpu.cu): the largest
   * s with max|J| * 2^s <= 2^23 - 1, J_int = rint(J * 2^s), bytes (u8, u8, s8). */
  float amax = 0.0f;
  for (int64_t k = 0; k < n * n; ++k) amax = fabsf(J[k]) > amax ? fabsf(J[k]) : amax;
  int shift = 0;
  while (ldexp((double)amax, shift + 1) <= 8388607.0 && shift < 60) ++shift;
  while (ldexp((double)amax, shift) > 8388607.0) --shift;
  for (int64_t k = 0; k < n * n; ++k) {
    const int32_t q = (int32_t)nearbyint(ldexp((double)J[k], shift));
    for (int a = 0; a < 3; ++a) planes[(int64_t)a * n * n + k] = (uint8_t)((uint32_t)q >> (8 * a));
  }
  return shift;
}

static inline int64_t jplane(const uint8_t* planes, int64_t n, int a, int64_t i, int64_t j) {
  const uint8_t b = planes[(int64_t)a * n * n + i * n + j];
  return a == 2 ? (int64_t)(int8_t)b : (int64_t)b;
}

void orc_fields_fx(int variant, int64_t n, const uint8_t* planes, int shift, int64_t R, int64_t ld, const float* x,
                   float* F) {
  /* The GPU's fixed-point field of real J (step_tma.cuh / step_pair.cuh, NA = 3) for R
   * replicas: F[r][i] = fl32(sum_w fl64(acc_w 2^(8w + e0))), acc_w = exact sum of the plane
   * products of weight w. */
  int64_t* qb = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * 4);
  for (int64_t r = 0; r < R; ++r) {
    const float* xr = x + r * ld;
    if (is_sign_variant(variant)) {
      for (int64_t j = 0; j < n; ++j) qb[j] = xr[j] >= 0.0f ? 1 : -1;
    } else {
      /* q = rint(x 2^30) as four SIGNED base-256 digits, the GPU's qdigits (gsb_phase.cuh) */
      for (int64_t j = 0; j < n; ++j) {
        const uint32_t u = (uint32_t)(quant30(xr[j]) + 0x00808080) ^ 0x00808080u;
        for (int b = 0; b < 4; ++b) qb[b * n + j] = (int64_t)(int8_t)(uint8_t)(u >> (8 * b));
      }
    }
    const int nb = is_sign_variant(variant) ? 1 : 4;
    const int nw = 3 + nb - 1;
    /* continuous variants: the plane products of weight 2^(8w), w = a + b < 2 (J's two low
     * bytes times q's two low digits, < 2^-27 of the field) are not formed (step_tma.cuh,
     * FX_W0): 9 of the 12 products */
    const int w0 = is_sign_variant(variant) ? 0 : 2;
    const int e0 = is_sign_variant(variant) ? -shift : -(shift + 30);
    for (int64_t i = 0; i < n; ++i) {
      int64_t acc[6] = {0, 0, 0, 0, 0, 0};
      for (int pa = 0; pa < 3; ++pa)
        for (int b = 0; b < nb; ++b) {
          if (pa + b < w0) continue;
          int64_t t = 0;
          for (int64_t j = 0; j < n; ++j) t += jplane(planes, n, pa, i, j) * qb[b * n + j];
          acc[pa + b] += t;
        }
      double f = 0.0;
      for (int w = w0; w < nw; ++w) f = f + (double)acc[w] * ldexp(1.0, 8 * w + e0);
      F[r * ld + i] = (float)f;
    }
  }
  free(qb);
}

void orc_step_f32_fx(int variant, int64_t n, const uint8_t* planes, int shift, int64_t R, int64_t ld, float* x,
                     float* y, float* p, uint64_t m, uint64_t M, float dt, float c, float a_cfg) {
  const float a = honours_a(variant) ? a_cfg : 0.0f;
  const float inv = 1.0f / (float)(M - m);
  float* F = (float*)malloc(sizeof(float) * (size_t)(R * ld));
  orc_fields_fx(variant, n, planes, shift, R, ld, x, F);
  for (int64_t r = 0; r < R; ++r)
    for (int64_t i = 0; i < n; ++i)
      orc_phase_f32(F[r * ld + i], x + r * ld + i, y + r * ld + i, p + r * ld + i, a, c, dt, inv);
  free(F);
}

void orc_energy2_fx(int64_t n, const uint8_t* planes, int64_t R, int64_t ld, const float* x, int64_t* E2) {
  /* exact sum_i s_i (J_int s)_i; energy = -E2/2 * 2^-shift */
  int8_t* s = (int8_t*)malloc((size_t)n);
  for (int64_t r = 0; r < R; ++r) {
    for (int64_t j = 0; j < n; ++j) s[j] = x[r * ld + j] >= 0.0f ? 1 : -1;
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) {
      int64_t field = 0;
      for (int64_t j = 0; j < n; ++j) {
        const int64_t q = jplane(planes, n, 0, i, j) + (jplane(planes, n, 1, i, j) << 8) + (jplane(planes, n, 2, i, j) << 16);
        field += q * s[j];
      }
      total += field * s[i];
    }
    E2[r] = total;
  }
  free(s);
}

/* Phase update over arrays with given fields (fields computed elsewhere, e.g. by a
 * row-sharded model); same op order as orc_phase_f32. */
void orc_phase_batch_f32(int64_t count, const float* F, float* x, float* y, float* p, float a, float c, float dt,
                         uint64_t m, uint64_t M) {
  const float inv = 1.0f / (float)(M - m);
  for (int64_t k = 0; k < count; ++k) orc_phase_f32(F[k], x + k, y + k, p + k, a, c, dt, inv);
}

/* Counter-based +-1 instance of sbg_gen_couplings_hash_pm1 (rows row0..row0+rows-1). */
void orc_gen_hash_pm1_rows(int64_t n, uint64_t seed, int64_t row0, int64_t rows, int8_t* Jr) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < n; ++j) {
      const int64_t i = row0 + r;
      int8_t v = 0;
      if (i != j) {
        const uint64_t lo = (uint64_t)(i < j ? i : j), hi = (uint64_t)(i < j ? j : i);
        v = (orc_mix64(seed ^ (lo * (uint64_t)n + hi)) >> 63) ? -1 : 1;
      }
      Jr[r * n + j] = v;
    }
}

void orc_init_reference_seeds(int64_t n, int64_t ld, int64_t R, const uint64_t* seeds, int chaos_probe, float* x,
                              float* y, float* p) {
  for (int64_t r = 0; r < R; ++r) { /* engine.cpp:25-39 with an explicit seed */
    xo_t g;
    xo_seed(&g, seeds[r]);
    for (int64_t i = 0; i < n; ++i)
      x[r * ld + i] = chaos_probe ? (float)(0.1 * xo_random_sign(&g)) : (float)xo_uniform_symmetric(&g);
    for (int64_t i = 0; i < n; ++i) {
      y[r * ld + i] = 0.0f;
      p[r * ld + i] = 1.0f;
    }
  }
}
