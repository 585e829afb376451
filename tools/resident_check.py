"""Resident-state kernel vs the streaming kernel: bitwise state equality, then timing."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402


def run(n, R, steps, variant, resident, a_rep=None):
    os.environ["SBG_RESIDENT"] = "1" if resident else "0"
    s = Solver(0)
    s.gen_random_dense(n, 1)
    s.init_state(R, InitMode.small_uniform, 1, 7)
    if a_rep is not None:
        s.set_replica_a(a_rep)
    cfg = SolverConfig(variant=Variant[variant], steps=1000, dt=1.25, c=1 / (2 * math.sqrt(n)), a=0.2)
    s.advance(cfg, 0, 3)
    s.synchronize()
    s.advance(cfg, 3, 3 + steps)
    ms = s.last_advance_ms()
    out = s.get_state()
    _, e, best, _ = s.readout()
    s.close()
    return out, e, ms


for n, R, steps, variant in [(300, 100, 7, "gdsb"), (2000, 1000, 10, "dsb"), (2000, 8192, 20, "gdsb"),
                             (1000, 3000, 9, "gdsb"), (4000, 512, 5, "gdsb")]:
    (a, ea, ta) = run(n, R, steps, variant, False)
    (b, eb, tb) = run(n, R, steps, variant, True)
    same = all((u.view(np.uint32) == v.view(np.uint32)).all() for u, v in zip(a, b)) and (ea == eb).all()
    print(f"n={n} R={R} {variant}: bitwise={same} stream {ta / steps * 1e3:.1f} us/step, "
          f"resident {tb / steps * 1e3:.1f} us/step", flush=True)
rng = np.random.default_rng(0)
arep = rng.random(700).astype(np.float32)
(a, ea, _), (b, eb, _) = run(500, 700, 6, "gdsb", False, arep), run(500, 700, 6, "gdsb", True, arep)
print("a_rep bitwise:", all((u.view(np.uint32) == v.view(np.uint32)).all() for u, v in zip(a, b)))
for steps in (200,):
    _, _, t = run(2000, 8192, steps, "gdsb", True)
    print(f"C2 resident {steps} steps: {t / steps * 1e3:.2f} us/step = {2000 * 8192 / (t / steps / 1e3):.3e} SU/s")
