"""profiles/r02_traffic.json from ncu launch lists of bench.py at two step counts.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size \
        --clock-control none --csv --log-file gpurun_out/r2_traffic_<K>.csv \
        python bench.py --steps <K> --warmup 5 --no-tts --no-cpu-baseline

For each config the TIMED advance of bench.py is picked out of the launch list (every
config runs a warm-up launch first, then the timed one) and its DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) recorded per launch of K steps. CSR (C3)
runs one csr_step_sm_kernel launch per replica slab and step: its entry sums the step
launches of the timed advance (the once-per-advance transposes are listed apart).
"""
import collections
import csv
import json
import sys

SPEC = {  # key: (kernel name as ncu prints it, which occurrence is the timed launch)
    "c2_resident_e2m1": ("void gsb_resident_ts_kernel<2, 4, 0, 0>", 1),
    "c1_planes": ("void gsb_multistep_pair_kernel<4, 64, 4, 2, 16, 0, 1, 0>", 1),
    "c4_sk": ("void gsb_multistep_pair_kernel<4, 128, 2, 2, 16, 0, 3, 0>", 1),
    "c5_single": ("void gsb_multistep_pair_kernel<1, 256, 5, 2, 16, 1, 1, 0>", 1),
}


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    idx = {x: j for j, x in enumerate(h)}
    out = collections.OrderedDict()
    for r in rows[i + 1:]:
        k = int(r[idx["ID"]])
        d = out.setdefault(k, {"name": r[idx["Kernel Name"]]})
        d[r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    return list(out.values())


def dram(d):
    return d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]


def main(files):
    res = {k: {"kernel": v[0], "launch_bytes": {}, "launch_ns": {}} for k, v in SPEC.items()}
    res["c3_csr"] = {"kernel": "csr_step_lean_kernel<0, 2> (one launch per replica slab and step, summed over the "
                               "timed advance)", "launch_bytes": {}, "launch_ns": {}, "transposes_bytes": {}}
    for f in files:
        K = int(f.rsplit("_", 1)[1].split(".")[0])
        L = launches(f)
        for key, (pref, occ) in SPEC.items():
            hits = [d for d in L if d["name"].startswith(pref)]
            d = hits[occ]
            res[key]["launch_bytes"][str(K)] = dram(d)
            res[key]["launch_ns"][str(K)] = d["gpu__time_duration.sum"]
        # C3: the CSR block after the (first) csr_prep_kernel; the state stays spin-major and the
        # operand current across advances, so the warm-up advance (W = 3 steps, one pass: no
        # slabs below 8 steps) and the timed one follow each other: the timed launches are the
        # block's step launches after the first 3
        preps = [i for i, d in enumerate(L) if d["name"].startswith("void csr_prep_kernel")]
        j = preps[0] + 1
        steps, trans = [], []
        while j < len(L) and (L[j]["name"].startswith("void csr_step") or L[j]["name"].startswith("transpose")):
            (steps if L[j]["name"].startswith("void csr_step") else trans).append(L[j])
            j += 1
        steps = steps[3:]
        res["c3_csr"]["launch_bytes"][str(K)] = sum(dram(d) for d in steps)
        res["c3_csr"]["launch_ns"][str(K)] = sum(d["gpu__time_duration.sum"] for d in steps)
        res["c3_csr"]["step_launches"] = res["c3_csr"].get("step_launches", {}) | {str(K): len(steps)}
        res["c3_csr"]["transposes_bytes"][str(K)] = sum(dram(d) for d in trans)
    res["_how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                   "--clock-control none on `python bench.py --steps K --warmup 5 --no-tts --no-cpu-baseline`, "
                   "K = " + ", ".join(sorted({f.rsplit('_', 1)[1].split('.')[0] for f in files})) +
                   "; the timed launch of each config; durations are serialised cold-cache ncu times")
    json.dump(res, open("profiles/r02_traffic.json", "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
