"""paper_2508_17655_b200 — B200-native generalized simulated bifurcation (GbSB/GdSB).

The hot path (the per-step GSB loop of sbopt::step, batched over replicas)
runs in hand-written sm_100a kernels behind the C ABI in include/sbgpu.h;
this package is the host-side mirror of the reference solver API.
"""
from .solver import (BatchResult, ConvergenceError, InitMode, SpectralEstimate, RunResult, Solver, SolverConfig, SuccessStats,  # noqa: F401
                     TtsResult, TuningResult, Variant, auto_tune_wigner, resolve_config,
                     success_from_counts, success_probability, success_probability_cut, time_to_solution)
from .instances import (CouplingEntries, CutGraph, ParseError, instance_from_json, instance_to_json,  # noqa: F401
                        load_gset, parse_gset, serialize_gset)
