"""Summarise an ncu report: key raw metrics + top stall SASS lines (run here, no GPU)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct",
        "sm__inst_executed_pipe_xu", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum ", "launch__grid_size", "sm__pipe_shared_cycles_active",
        "l1tex__throughput.avg.pct", "dram__throughput.avg.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:] if len(rows) > 2 else rows[1:]


def main(rep, top=25):
    h, data = raw(rep)
    for v in data:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("kernel:", name[:100])
        for k, x in zip(h, v):
            if any(k.startswith(w.strip()) or w.strip() == k for w in KEYS):
                print(f"  {k} = {x}")
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    body = rows[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    tot = sum(float(r[iS] or 0) for r in body) or 1
    print(f"stall samples: {tot:.0f}")
    for r in sorted(body, key=lambda r: -float(r[iS] or 0))[:top]:
        print(f"  {100 * float(r[iS]) / tot:5.1f}% {r[iE]:>10} {r[1][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
