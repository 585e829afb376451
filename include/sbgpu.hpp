// sbgpu.hpp — header-only C++ mirror of the reference solver API over the C ABI.
//
// Same names, fields and error behaviour as sbopt (/root/reference/proj/core/include/sbopt/
// engine.hpp:26-64, bench.hpp:22-67, spectral.hpp:28-33), so code written against
// sbopt::run / batch_best_of / success_probability / time_to_solution moves over
// by namespace. Argument errors surface as std::invalid_argument exactly where the
// reference throws them (engine.cpp:16-21, :57-60; model.cpp:56-66; bench.cpp:16-17,
// :53-54); device/runtime failures as std::runtime_error. Nothing here computes
// the hot path: every step runs in libsbgpu.so's sm_100a kernels.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sbgpu.h"

namespace sbgpu {

enum class Variant { bsb = SBG_BSB, dsb = SBG_DSB, gbsb = SBG_GBSB, gdsb = SBG_GDSB };
enum class InitMode {
  uniform_random = SBG_INIT_UNIFORM_RANDOM,
  chaos_probe = SBG_INIT_CHAOS_PROBE,
  small_uniform = SBG_INIT_SMALL_UNIFORM
};

namespace seed_stream {  // rng.hpp:33-40 (+ the BASELINE device-init stream)
inline constexpr std::uint64_t batch = 3;
inline constexpr std::uint64_t gpu_init = 7;
}  // namespace seed_stream

struct SolverConfig {  // engine.hpp:29-38
  Variant variant = Variant::gbsb;
  std::uint64_t steps = 1000;
  std::optional<double> dt;
  std::optional<double> c;
  double a = 0.0;
  std::uint64_t seed = 0;
  InitMode init_mode = InitMode::uniform_random;
};

enum class SpectralMethod {  // spectral.hpp:17
  power_iteration = SBG_SPECTRAL_POWER_ITERATION,
  wigner = SBG_SPECTRAL_WIGNER,
  exact_small = SBG_SPECTRAL_EXACT_SMALL
};
enum class TuneMode { wigner = SBG_TUNE_WIGNER, numerical = SBG_TUNE_NUMERICAL };  // spectral.hpp:64

struct SpectralEstimate {  // spectral.hpp:19-27
  double lambda_max = 0.0;
  double lambda_min = 0.0;
  SpectralMethod method = SpectralMethod::power_iteration;
  double tolerance = 0.0;
  std::vector<double> v_max;  // empty for wigner
  std::vector<double> v_min;
  std::size_t iterations = 0;
};

// spectral.hpp:38-47: estimation missed the residual target; best estimate attached.
class ConvergenceError : public std::runtime_error {
 public:
  ConvergenceError(const std::string& message, SpectralEstimate last)
      : std::runtime_error(message), last_(std::move(last)) {}
  const SpectralEstimate& last_estimate() const noexcept { return last_; }

 private:
  SpectralEstimate last_;
};

struct TuningResult {  // spectral.hpp:28-33 (lambda_max/lambda_min mirror source's edges)
  double c = 0.0;
  double dt = 0.0;
  double d_t_factor = 0.0;
  double lambda_max = 0.0;
  double lambda_min = 0.0;
  SpectralEstimate source;
};

struct RunResult {  // engine.hpp:56-64
  std::vector<std::int8_t> final_spins;
  double energy = 0.0;
  std::optional<long long> cut;
  double wall_time_s = 0.0;
  SolverConfig config_echo;
  TuningResult tuning_echo;
};

struct SuccessStats {  // bench.hpp:22-28
  double p_s = 0.0;
  double delta_p_s = 0.0;
  std::size_t n_rep = 0;
  double target_value = 0.0;
  std::size_t hit_count = 0;
};

struct TtsResult {  // bench.hpp:41-46
  double tts_s = 0.0;
  double delta_tts_s = 0.0;
  double t_com_s = 0.0;
  SuccessStats stats;
};

namespace detail {
inline void check(int rc, const char* msg) {
  if (rc == SBG_OK) return;
  if (rc == SBG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg ? msg : "invalid argument");
  throw std::runtime_error(std::string("sbgpu: ") + sbg_strerror(rc) + (msg ? std::string(": ") + msg : ""));
}
constexpr std::uint64_t mix64(std::uint64_t z) noexcept {  // rng.hpp:17-21
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
}  // namespace detail

// rng.hpp:26-31 (used for config echoes; device seeds are derived on the GPU).
inline std::uint64_t derive_seed(std::uint64_t master, std::initializer_list<std::uint64_t> keys) noexcept {
  std::uint64_t h = detail::mix64(master + 0x9E3779B97F4A7C15ULL);
  for (std::uint64_t k : keys) h = detail::mix64(h ^ (k + 0x9E3779B97F4A7C15ULL));
  return h;
}

// resolve_config + validate (engine.cpp:16-21, :48-53).
inline SolverConfig resolve_config(SolverConfig cfg, const TuningResult& tuning) {
  if (!cfg.dt) cfg.dt = tuning.dt;
  if (!cfg.c) cfg.c = tuning.c;
  if (cfg.steps < 1) throw std::invalid_argument("step count M must be >= 1");
  if (!(*cfg.dt > 0.0)) throw std::invalid_argument("dt must be positive");
  if (!(*cfg.c > 0.0)) throw std::invalid_argument("c must be positive");
  if (!(cfg.a >= 0.0)) throw std::invalid_argument("A must be >= 0");
  return cfg;
}

inline SuccessStats success_from_counts(std::size_t hit_count, std::size_t n_rep, double target) {
  if (n_rep == 0) throw std::invalid_argument("success probability needs n_rep >= 1");
  if (hit_count > n_rep) throw std::invalid_argument("hit count exceeds repetitions");
  double out[4];
  sbg_success_tts(static_cast<std::int64_t>(hit_count), static_cast<std::int64_t>(n_rep), 1.0, out);
  return SuccessStats{out[0], out[1], n_rep, target, hit_count};
}

// bench.cpp:28-36 (energy_min hit rule: energy <= target, exact).
inline SuccessStats success_probability(const std::vector<double>& energies, double target) {
  if (energies.empty()) throw std::invalid_argument("no results");
  std::size_t hits = 0;
  for (double e : energies)
    if (e <= target) ++hits;
  return success_from_counts(hits, energies.size(), target);
}

inline TtsResult time_to_solution(double t_com_s, const SuccessStats& stats) {  // bench.cpp:52-68
  if (!(t_com_s > 0.0)) throw std::invalid_argument("t_com must be positive");
  if (!(stats.p_s > 0.0)) throw std::invalid_argument("TTS undefined for p_s = 0");
  double out[4];
  detail::check(sbg_success_tts(static_cast<std::int64_t>(stats.hit_count), static_cast<std::int64_t>(stats.n_rep),
                                t_com_s, out),
                "time_to_solution");
  return TtsResult{out[2], out[3], t_com_s, stats};
}

// auto_tune(TuneMode::wigner) on a dense fp64 instance (spectral.cpp:294-326).
inline TuningResult auto_tune_wigner(std::size_t n, const std::vector<double>& J, double d_t_factor = 1.25) {
  TuningResult t;
  t.d_t_factor = d_t_factor;
  detail::check(sbg_tune_wigner_f64(static_cast<std::int64_t>(n), J.data(), d_t_factor, &t.c, &t.dt),
                "degenerate instance: all couplings zero");
  t.lambda_max = 1.0 / t.c;
  t.lambda_min = -t.lambda_max;
  return t;
}

// One device context: the batched replacement for run() / batch_best_of().
class Solver {
 public:
  explicit Solver(int device = 0) {
    const int rc = sbg_create(device, &ctx_);
    if (rc != SBG_OK) detail::check(rc == SBG_ERR_INVALID_ARGUMENT ? rc : rc, "sbg_create failed");
  }
  ~Solver() { sbg_destroy(ctx_); }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  // IsingInstance (model.hpp:46-70) as stored by the reference: dense row-major fp64.
  void set_instance(std::size_t n, const std::vector<double>& J, std::optional<long long> total_weight = {}) {
    if (J.size() != n * n) throw std::invalid_argument("coupling matrix must have n*n entries");
    check(sbg_set_couplings_dense_f64(ctx_, static_cast<std::int64_t>(n), J.data()));
    n_ = n;
    if (total_weight) {
      total_weight_ = total_weight;
    } else {  // dense instance without a graph: w = -J (model.hpp:103-104)
      long long w = 0;
      for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = i + 1; j < n; ++j) w -= static_cast<long long>(J[i * n + j]);
      total_weight_ = w;
    }
  }
  void set_instance_i8(std::size_t n, const std::int8_t* J) {
    check(sbg_set_couplings_dense_i8(ctx_, static_cast<std::int64_t>(n), J));
    n_ = n;
    long long w = 0;
    for (std::size_t i = 0; i < n; ++i)
      for (std::size_t j = i + 1; j < n; ++j) w -= J[i * n + j];
    total_weight_ = w;
  }
  // gen_random_dense (model.cpp:144-159) evaluated straight into the device instance.
  void gen_random_dense(std::size_t n, std::uint64_t seed) {
    check(sbg_gen_couplings_dense_pm1(ctx_, static_cast<std::int64_t>(n), seed));
    n_ = n;
    total_weight_.reset();
  }

  // extreme_eigenvalues (spectral.cpp:207-246) of the device couplings.
  SpectralEstimate extreme_eigenvalues(double tol = 1e-6, std::size_t max_iters = 0) {
    sbg_spectral st{};
    SpectralEstimate e;
    e.v_max.resize(n_);
    e.v_min.resize(n_);
    const int rc = sbg_extreme_eigenvalues(ctx_, tol, max_iters, &st, e.v_max.data(), e.v_min.data());
    fill(st, e);
    if (rc == SBG_ERR_CONVERGENCE) throw ConvergenceError(sbg_last_error(ctx_), e);
    check(rc);
    return e;
  }
  // auto_tune (spectral.cpp:294-326) of the device couplings.
  TuningResult auto_tune(TuneMode mode, double d_t_factor = 1.25, double tol = 1e-6, std::size_t max_iters = 0) {
    sbg_spectral st{};
    const int rc = sbg_auto_tune(ctx_, static_cast<std::int32_t>(mode), d_t_factor, tol, max_iters, &st);
    TuningResult t;
    fill(st, t.source);
    if (rc == SBG_ERR_CONVERGENCE) throw ConvergenceError(sbg_last_error(ctx_), t.source);
    check(rc);
    t.c = st.c;
    t.dt = st.dt;
    t.d_t_factor = st.d_t_factor;
    t.lambda_max = st.lambda_max;
    t.lambda_min = st.lambda_min;
    return t;
  }

  // R runs of run() (engine.cpp:112-139) in one device pass; replica r is seeded
  // derive_seed(master_seed, {tag, r}) with cfg.init_mode. Returns one RunResult per
  // replica (final spins, energy, cut when a total weight is known).
  std::vector<RunResult> run_batch(const SolverConfig& cfg, const TuningResult& tuning, std::size_t R,
                                   std::uint64_t master_seed, std::uint64_t tag = seed_stream::batch) {
    const SolverConfig rc = resolve_config(cfg, tuning);
    const sbg_params prm = params(rc);
    std::vector<std::int8_t> spins(R * n_);
    std::vector<double> energy(R);
    std::int64_t best = 0;
    sbg_timing timing{};
    const auto t0 = std::chrono::steady_clock::now();
    check(sbg_run_seeded(ctx_, &prm, static_cast<std::int64_t>(R), static_cast<std::int32_t>(rc.init_mode),
                         master_seed, tag, 0, spins.data(), energy.data(), &best, &timing));
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<RunResult> out(R);
    for (std::size_t r = 0; r < R; ++r) {
      RunResult& res = out[r];
      res.final_spins.assign(spins.begin() + static_cast<std::ptrdiff_t>(r * n_),
                             spins.begin() + static_cast<std::ptrdiff_t>((r + 1) * n_));
      res.energy = energy[r];
      if (total_weight_) res.cut = (*total_weight_ - static_cast<long long>(energy[r])) / 2;
      res.wall_time_s = wall;
      res.config_echo = rc;
      res.config_echo.seed = derive_seed(master_seed, {tag, static_cast<std::uint64_t>(r)});
      res.tuning_echo = tuning;
    }
    last_best_ = static_cast<std::size_t>(best);
    return out;
  }

  // bench.cpp:70-92: min energy, ties to the lowest replica index; wall time of the batch.
  RunResult batch_best_of(const SolverConfig& cfg, const TuningResult& tuning, std::size_t n_batch,
                          std::uint64_t master_seed) {
    if (n_batch < 1) throw std::invalid_argument("batch size must be >= 1");
    auto all = run_batch(cfg, tuning, n_batch, master_seed, seed_stream::batch);
    return std::move(all[last_best_]);
  }

  // batch_best_of from host initial states (x0, y0: R x n, replica-major) in one device pass
  // (sbg_run_best): only the winner -- its spins, energy and index (ties to the lowest
  // replica, bench.cpp:84-87) -- crosses back to the host. best_index receives the index.
  RunResult batch_best_of_states(const SolverConfig& cfg, const TuningResult& tuning, std::size_t R,
                                 const std::vector<float>& x0, const std::vector<float>& y0,
                                 std::size_t* best_index = nullptr) {
    if (R < 1) throw std::invalid_argument("batch size must be >= 1");
    if (x0.size() != R * n_ || y0.size() != R * n_) throw std::invalid_argument("initial state size mismatch");
    const SolverConfig rc = resolve_config(cfg, tuning);
    const sbg_params prm = params(rc);
    RunResult res;
    res.final_spins.resize(n_);
    std::int64_t best = 0;
    sbg_timing timing{};
    check(sbg_run_best(ctx_, &prm, static_cast<std::int64_t>(R), x0.data(), y0.data(), res.final_spins.data(),
                       &res.energy, &best, nullptr, &timing));
    if (total_weight_) res.cut = (*total_weight_ - static_cast<long long>(res.energy)) / 2;
    res.wall_time_s = timing.total_ms / 1e3;
    res.config_echo = rc;
    res.tuning_echo = tuning;
    if (best_index) *best_index = static_cast<std::size_t>(best);
    return res;
  }

  std::size_t n() const noexcept { return n_; }
  sbg_ctx* handle() noexcept { return ctx_; }

 private:
  static sbg_params params(const SolverConfig& c) {
    sbg_params p{};
    p.variant = static_cast<std::int32_t>(c.variant);
    p.steps = c.steps;
    p.dt = *c.dt;
    p.c = *c.c;
    p.a = c.a;
    return p;
  }
  void check(int rc) const { detail::check(rc, sbg_last_error(ctx_)); }
  static void fill(const sbg_spectral& st, SpectralEstimate& e) {
    e.lambda_max = st.lambda_max;
    e.lambda_min = st.lambda_min;
    e.method = static_cast<SpectralMethod>(st.method);
    e.tolerance = st.tolerance;
    e.iterations = static_cast<std::size_t>(st.iterations);
    if (e.method == SpectralMethod::wigner) {
      e.v_max.clear();
      e.v_min.clear();
    }
  }

  sbg_ctx* ctx_ = nullptr;
  std::size_t n_ = 0;
  std::optional<long long> total_weight_;
  std::size_t last_best_ = 0;
};

}  // namespace sbgpu
