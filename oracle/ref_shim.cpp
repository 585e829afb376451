// TEST INFRASTRUCTURE ONLY. Never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference core library (sbopt, compiled
// from /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/). It exposes exactly the reference entry points the parity
// tests and the bench's reference arm need, with plain pointers so Python can
// call them through ctypes. Nothing here re-implements the algorithm: every
// numeric result comes from the reference's own step()/run()/coupling_matvec()
// /ising_energy()/batch_best_of()/auto_tune()/time_to_solution().
//
// Reference interfaces wrapped (paths relative to /root/reference/proj/core):
//   step                 src/engine.cpp:55-110   (include/sbopt/engine.hpp:79-80)
//   init_state           src/engine.cpp:25-39
//   run                  src/engine.cpp:112-139
//   coupling_matvec      src/kernels.hpp:33-46
//   ising_energy         src/model.cpp:112-123
//   gen_random_dense     src/model.cpp:144-159
//   auto_tune (wigner)   src/spectral.cpp:294-326
//   batch_best_of        src/bench.cpp:70-92
//   success/TTS          src/bench.cpp:15-68
//   ThreadPool           src/parallel.cpp:59-84

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "sbopt/bench.hpp"
#include "sbopt/chaos.hpp"
#include "sbopt/engine.hpp"
#include "sbopt/model.hpp"
#include "sbopt/parallel.hpp"
#include "sbopt/rng.hpp"
#include "sbopt/spectral.hpp"

using namespace sbopt;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

Variant to_variant(int v) {
  switch (v) {
    case 0: return Variant::bsb;
    case 1: return Variant::dsb;
    default: return Variant::gbsb;
  }
}

IsingInstance make_instance(std::int64_t n, const double* J) {
  return IsingInstance(static_cast<std::size_t>(n),
                       std::vector<double>(J, J + static_cast<std::size_t>(n * n)));
}

SolverConfig make_cfg(int variant, std::uint64_t steps, double dt, double c, double a,
                      std::uint64_t seed) {
  SolverConfig cfg;
  cfg.variant = to_variant(variant);
  cfg.steps = steps;
  cfg.dt = dt;
  cfg.c = c;
  cfg.a = a;
  cfg.seed = seed;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_derive_seed(std::uint64_t master, const std::uint64_t* keys, int nkeys) {
  // derive_seed takes an initializer_list; fold the same way for 0..3 keys.
  switch (nkeys) {
    case 0: return derive_seed(master, {});
    case 1: return derive_seed(master, {keys[0]});
    case 2: return derive_seed(master, {keys[0], keys[1]});
    default: return derive_seed(master, {keys[0], keys[1], keys[2]});
  }
}

void ref_xoshiro_next(std::uint64_t seed, std::int64_t count, std::uint64_t* out) {
  Xoshiro256pp rng(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = rng.next();
}

int ref_gen_random_dense(std::int64_t n, std::uint64_t seed, double* J_out) {
  try {
    const auto inst = gen_random_dense(static_cast<std::size_t>(n), seed);
    for (std::int64_t i = 0; i < n; ++i) {
      const auto row = inst.row(static_cast<std::size_t>(i));
      std::memcpy(J_out + i * n, row.data(), sizeof(double) * static_cast<std::size_t>(n));
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_init_state(std::int64_t n, std::uint64_t seed, int chaos_probe, double* x, double* y,
                   double* p) {
  try {
    const auto s = init_state(static_cast<std::size_t>(n), seed,
                              chaos_probe ? InitMode::chaos_probe : InitMode::uniform_random);
    std::memcpy(x, s.x.data(), sizeof(double) * s.x.size());
    std::memcpy(y, s.y.data(), sizeof(double) * s.y.size());
    std::memcpy(p, s.p.data(), sizeof(double) * s.p.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Advances an injected state (x, y, p at step index m0) by nsteps calls of the
// reference step(). BASELINE initial states are not producible by run()
// (engine.cpp:25-39 always draws x ~ U(-1,1)), so the harness builds the
// SolverState itself and replicates run()'s loop (engine.cpp:121-126).
int ref_step_n(int variant, std::int64_t n, const double* J, double* x, double* y, double* p,
               std::uint64_t m0, std::uint64_t steps, double dt, double c, double a,
               std::uint64_t nsteps) {
  try {
    const auto inst = make_instance(n, J);
    const auto cfg = make_cfg(variant, steps, dt, c, a, 0);
    SolverState s;
    s.x.assign(x, x + n);
    s.y.assign(y, y + n);
    s.p.assign(p, p + n);
    s.m = m0;
    for (std::uint64_t k = 0; k < nsteps; ++k) step(s, inst, cfg, nullptr);
    std::memcpy(x, s.x.data(), sizeof(double) * static_cast<std::size_t>(n));
    std::memcpy(y, s.y.data(), sizeof(double) * static_cast<std::size_t>(n));
    std::memcpy(p, s.p.data(), sizeof(double) * static_cast<std::size_t>(n));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_coupling_matvec(std::int64_t n, const double* J, const double* v, double* out) {
  try {
    const auto inst = make_instance(n, J);
    detail::coupling_matvec(inst, v, out, nullptr);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_ising_energy(std::int64_t n, const double* J, const std::int8_t* spins, double* energy) {
  try {
    const auto inst = make_instance(n, J);
    *energy = ising_energy(inst, SpinConfig(std::vector<std::int8_t>(spins, spins + n)));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_auto_tune_wigner(std::int64_t n, const double* J, double d_t, double* c, double* dt) {
  try {
    const auto t = auto_tune(make_instance(n, J), TuneMode::wigner, d_t);
    *c = t.c;
    *dt = t.dt;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// run() with the reference's own init (engine.cpp:112-139).
int ref_run(int variant, std::int64_t n, const double* J, std::uint64_t steps, double dt,
            double c, double a, std::uint64_t seed, std::int8_t* spins, double* energy,
            double* x_final_unused) {
  (void)x_final_unused;
  try {
    const auto inst = make_instance(n, J);
    TuningResult t;
    t.c = c;
    t.dt = dt;
    const auto r = run(inst, make_cfg(variant, steps, dt, c, a, seed), t, nullptr, nullptr);
    std::memcpy(spins, r.final_spins.values().data(), static_cast<std::size_t>(n));
    *energy = r.energy;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_batch_best_of(int variant, std::int64_t n, const double* J, std::uint64_t steps, double dt,
                      double c, double a, std::int64_t n_batch, std::uint64_t master,
                      unsigned workers, std::int8_t* spins, double* energy,
                      std::uint64_t* seed_out) {
  try {
    const auto inst = make_instance(n, J);
    TuningResult t;
    t.c = c;
    t.dt = dt;
    const auto r = batch_best_of(inst, make_cfg(variant, steps, dt, c, a, 0), t,
                                 static_cast<std::size_t>(n_batch), master, workers, nullptr);
    std::memcpy(spins, r.final_spins.values().data(), static_cast<std::size_t>(n));
    *energy = r.energy;
    *seed_out = r.config_echo.seed;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_success_tts(std::int64_t hits, std::int64_t n_rep, double t_com, double* p_s,
                    double* delta_p_s, double* tts, double* delta_tts) {
  try {
    const auto st = success_from_counts(static_cast<std::size_t>(hits),
                                        static_cast<std::size_t>(n_rep), 0.0);
    *p_s = st.p_s;
    *delta_p_s = st.delta_p_s;
    const auto tr = time_to_solution(t_com, st);
    *tts = tr.tts_s;
    *delta_tts = tr.delta_tts_s;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference arm of the bench: cmd_bench's replica fan-out
// (tools/sbopt.cpp:265-272) over injected initial states. R replicas are
// distributed with ThreadPool::for_each_index; each replica runs `steps`
// reference step() calls (pool = nullptr, as bench.cpp:81 does), then
// signs_from_positions + ising_energy. x0/y0 are R x n fp32 (BASELINE init),
// widened to fp64. Returns wall seconds of the whole fan-out.
int ref_replica_fanout(int variant, std::int64_t n, const double* J, std::int64_t R,
                       const float* x0, const float* y0, std::uint64_t steps, double dt, double c,
                       double a, unsigned workers, double* energies, double* wall_s) {
  try {
    const auto inst = make_instance(n, J);
    const auto cfg = make_cfg(variant, steps, dt, c, a, 0);
    ThreadPool pool(workers);
    const auto t0 = std::chrono::steady_clock::now();
    pool.for_each_index(static_cast<std::size_t>(R), [&](std::size_t r) {
      SolverState s;
      s.x.assign(x0 + r * n, x0 + (r + 1) * n);
      s.y.assign(y0 + r * n, y0 + (r + 1) * n);
      s.p.assign(static_cast<std::size_t>(n), 1.0);
      s.m = 0;
      for (std::uint64_t m = 0; m < steps; ++m) step(s, inst, cfg, nullptr);
      energies[r] = ising_energy(inst, signs_from_positions(s.x));
    });
    *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

unsigned ref_effective_workers(unsigned requested) { return effective_workers(requested); }

// parse_gset (model.cpp:225-282). Returns 0 and fills n, m (and up to cap edges as
// 0-based i, j, w); 2 on ParseError / invalid_argument with the message in ref_last_error.
int ref_parse_gset(const char* text, std::int64_t* n, std::int64_t* m, std::int64_t cap, std::int64_t* ei,
                   std::int64_t* ej, std::int64_t* w) {
  try {
    const auto g = parse_gset(std::string_view(text));
    *n = static_cast<std::int64_t>(g.n());
    *m = static_cast<std::int64_t>(g.edges().size());
    std::int64_t k = 0;
    for (const auto& e : g.edges()) {
      if (k >= cap) break;
      ei[k] = static_cast<std::int64_t>(e.i);
      ej[k] = static_cast<std::int64_t>(e.j);
      w[k] = e.w;
      ++k;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// cut_value (model.cpp:125-132) of a CutGraph for given spins.
int ref_cut_value(std::int64_t n, std::int64_t m, const std::int64_t* ei, const std::int64_t* ej,
                  const std::int64_t* w, const std::int8_t* spins, long long* cut) {
  try {
    std::vector<CutEdge> edges;
    edges.reserve(static_cast<std::size_t>(m));
    for (std::int64_t k = 0; k < m; ++k)
      edges.push_back({static_cast<std::size_t>(ei[k]), static_cast<std::size_t>(ej[k]), w[k]});
    const CutGraph g(static_cast<std::size_t>(n), std::move(edges));
    *cut = cut_value(g, SpinConfig(std::vector<std::int8_t>(spins, spins + n)));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// instance_from_json (model.cpp:318-348) -> dense fp64 (n*n must fit J_out's cap).
int ref_instance_from_json(const char* text, std::int64_t cap, std::int64_t* n, double* J_out) {
  try {
    const auto inst = instance_from_json(std::string_view(text));
    *n = static_cast<std::int64_t>(inst.n());
    if (*n * *n <= cap)
      for (std::int64_t i = 0; i < *n; ++i) {
        const auto row = inst.row(static_cast<std::size_t>(i));
        std::memcpy(J_out + i * *n, row.data(), sizeof(double) * static_cast<std::size_t>(*n));
      }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

// instance_to_json (model.cpp:296-316) of a dense fp64 instance; returns the length
// written (truncated at cap - 1) or -1.
std::int64_t ref_instance_to_json(std::int64_t n, const double* J, char* out, std::int64_t cap) {
  try {
    const auto s = instance_to_json(make_instance(n, J));
    const auto len = std::min<std::int64_t>(static_cast<std::int64_t>(s.size()), cap - 1);
    std::memcpy(out, s.data(), static_cast<std::size_t>(len));
    out[len] = 0;
    return static_cast<std::int64_t>(s.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// extreme_eigenvalues (spectral.cpp:207-246). out6 = {lambda_max, lambda_min,
// iterations, method, tolerance, converged}; v_max / v_min n doubles (or null).
// Returns 0, 1 (invalid argument) or 7 (ConvergenceError, carried estimate in out6).
int ref_extreme_eigenvalues(std::int64_t n, const double* J, double tol, std::uint64_t max_iters, double* out6,
                            double* v_max, double* v_min) {
  auto fill = [&](const SpectralEstimate& e, bool conv) {
    out6[0] = e.lambda_max;
    out6[1] = e.lambda_min;
    out6[2] = static_cast<double>(e.iterations);
    out6[3] = static_cast<double>(static_cast<int>(e.method));
    out6[4] = e.tolerance;
    out6[5] = conv ? 1.0 : 0.0;
    if (v_max && e.v_max.size() == static_cast<std::size_t>(n)) std::memcpy(v_max, e.v_max.data(), sizeof(double) * n);
    if (v_min && e.v_min.size() == static_cast<std::size_t>(n)) std::memcpy(v_min, e.v_min.data(), sizeof(double) * n);
  };
  try {
    fill(extreme_eigenvalues(make_instance(n, J), tol, static_cast<std::size_t>(max_iters)), true);
    return 0;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    fill(e.last_estimate(), false);
    return 7;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// auto_tune (spectral.cpp:294-326): out4 = {c, dt, lambda_max, lambda_min}.
int ref_auto_tune(std::int64_t n, const double* J, int numerical, double d_t, double tol, std::uint64_t max_iters,
                  double* out4) {
  try {
    const auto t = auto_tune(make_instance(n, J), numerical ? TuneMode::numerical : TuneMode::wigner, d_t, tol,
                             static_cast<std::size_t>(max_iters));
    out4[0] = t.c;
    out4[1] = t.dt;
    out4[2] = t.source.lambda_max;
    out4[3] = t.source.lambda_min;
    return 0;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// chaos_scan (chaos.cpp:65-102): final deltas, row-major [a][rep].
int ref_chaos_scan(std::int64_t n, const double* J, const double* a_values, std::int64_t na, std::int64_t reps,
                   std::uint64_t steps, double dt, double c, std::uint64_t seed, unsigned workers,
                   double* final_deltas) {
  try {
    const auto inst = make_instance(n, J);
    TuningResult t;
    t.c = c;
    t.dt = dt;
    SolverConfig cfg = make_cfg(2, steps, dt, c, 0.0, seed);
    const auto rows = chaos_scan(inst, std::span<const double>(a_values, static_cast<std::size_t>(na)),
                                 static_cast<std::size_t>(reps), cfg, t, workers);
    for (std::size_t ai = 0; ai < rows.size(); ++ai)
      for (std::size_t r = 0; r < rows[ai].final_deltas.size(); ++r)
        final_deltas[ai * static_cast<std::size_t>(reps) + r] = rows[ai].final_deltas[r];
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
