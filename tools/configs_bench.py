"""Per-config throughput of the hot path for the BASELINE configs C1..C4 (one GPU).

C1 N=2000 dense +-1 GbSB R=1000 | C2 GdSB R=8192 | C3 ER N=20000 d=10 CSR GbSB R=512
| C4 SK N=4096 GbSB R=2048. Timed: K steps after a warm-up launch, device events.
"""
import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (instance generators only; the timed path is the GPU)
from paper_2508_17655_b200 import InitMode, Solver, SolverConfig, Variant  # noqa: E402

HBM = 6553.0
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def peak(name, key):
    """Measured tensor peaks (profiles/int8_peak.json, profiles/fp4_peak.json), TOP/s."""
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return float(json.load(f)[key])


def run(s, variant, n, R, steps, c, bytes_per_su_extra=0.0, ops_per_su=None, tensor_peak=None):
    cfg = SolverConfig(variant=variant, steps=1000 + steps, dt=1.25, c=c, a=0.2)
    s.init_state(R, InitMode.small_uniform, 1, 7)
    s.advance(cfg, 0, 3)
    s.synchronize()
    s.advance(cfg, 3, 3 + steps)
    ms = s.last_advance_ms()
    us = ms / steps * 1e3
    su = n * R / (us * 1e-6)
    out = {"us_per_step": us, "su_per_s": su}
    b = (24 + bytes_per_su_extra) * n * R
    out["gbs"] = b / (us * 1e-6) / 1e9
    out["hbm_frac"] = out["gbs"] / HBM
    if ops_per_su:
        out["tops"] = ops_per_su * n * R / (us * 1e-6) / 1e12
        if tensor_peak:
            out["tensor_frac"] = out["tops"] / tensor_peak[0]
            out["tensor_peak"] = tensor_peak[1]
    # the sign variants multiply with kind::mxf4 when J has an e2m1 copy; bSB/GbSB use int8 planes
    sign = variant in (Variant.dsb, Variant.gdsb)
    out["mma"] = "kind::mxf4 (e2m1)" if sign and s.operand_format == "e2m1" else "kind::i8"
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--only", default="C1,C2,C3,C4")
    args = ap.parse_args()
    orc = oracle.orc()
    res = {}
    i8 = (peak("int8_peak.json", "int8_tops_burst"), "int8 (cuBLASLt 8192^3 burst)")
    f4 = (peak("fp4_peak.json", "fp4_tops_burst"), "fp4 (cuBLASLt NVFP4 8192^3 burst)")
    with Solver(0) as s:
        only = args.only.split(",")
        if "C1" in only or "C2" in only:
            s.gen_random_dense(2000, 1)
            c = 1 / (2 * math.sqrt(2000))
            if "C1" in only:
                res["C1_gbsb_n2000_R1000"] = run(s, Variant.gbsb, 2000, 1000, args.steps, c, 2000 / 1000,
                                                 ops_per_su=4 * 2 * 2000, tensor_peak=i8)
            if "C2" in only:
                res["C2_gdsb_n2000_R8192"] = run(s, Variant.gdsb, 2000, 8192, args.steps, c, 2000 / 8192,
                                                 ops_per_su=2 * 2000, tensor_peak=f4)
        if "C3" in only:
            n, m = 20000, 100000
            _, (rowptr, col, val) = orc.gen_er_csr(n, m, 1)
            s.set_instance_csr(n, rowptr, col, val)
            c = 1 / (2 * math.sqrt(n) * math.sqrt(2 * m / (n * (n - 1))))  # Wigner on the dense view
            csr_bytes = (4 * (n + 1) + 5 * 2 * m) / (n * 512)  # CSR once per step
            res["C3_gbsb_er_n20000_R512"] = run(s, Variant.gbsb, n, 512, args.steps, c, csr_bytes)
            res["C3_gbsb_er_n20000_R512"]["c"] = c
            res["C3_gbsb_er_n20000_R512"]["mma"] = "CSR SIMT (exact int64)"
        if "C4" in only:
            n = 4096
            J = orc.gen_sk_f32(n, 1)
            s.set_instance(J)
            res["C4_gbsb_sk_n4096_R2048"] = run(s, Variant.gbsb, n, 2048, args.steps, 0.5, 3 * n / 2048,
                                                ops_per_su=9 * 2 * n, tensor_peak=i8)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
