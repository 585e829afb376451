"""Times the bench's TTS leg shape (N=2000, 1000 runs, M=21500, reference init) for one variant,
and the bare advance of the same length (dev A/B of the resident kernel choice)."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, TuningResult, Variant  # noqa: E402

v = sys.argv[1] if len(sys.argv) > 1 else "gdsb"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 21500
R = int(sys.argv[3]) if len(sys.argv) > 3 else 1000
s = Solver(0)
s.gen_random_dense(2000, 1)
c = 1 / (2 * math.sqrt(2000))
cfg = SolverConfig(variant=Variant[v], steps=M, dt=1.25, c=c, a=0.2, init_mode=InitMode.uniform_random)
tun = TuningResult(c=c, dt=1.25)
s.run_batch(cfg, tun, 64, master_seed=7, want_spins=False)
for rep in range(3):
    t0 = time.perf_counter()
    b = s.run_batch(cfg, tun, R, master_seed=1, want_spins=False)
    t = time.perf_counter() - t0
    print(f"{v} run_batch R={R} M={M}: {t * 1e3:.1f} ms wall, device {b.timing['total_ms']:.1f} ms "
          f"({b.timing['total_ms'] / M * 1e3:.2f} us/step), init {b.timing['init_ms']:.1f} steps {b.timing['steps_ms']:.1f}")
s.init_state(R, InitMode.uniform_random, 1, 3)
s.advance(cfg, 0, 50)
s.synchronize()
s.advance(cfg, 50, M)
s.synchronize()
ms = s.last_advance_ms()
print(f"{v} advance R={R} steps={M - 50}: {ms / (M - 50) * 1e3:.2f} us/step")
s.close()
