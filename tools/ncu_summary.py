"""Summarise an ncu --set full report: headline metrics + top stall sites (SASS)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L2 Cache Throughput", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy", "No Eligible",
        "Active Warps Per Scheduler", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Registers Per Thread", "Achieved Occupancy", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Avg. Active Threads Per Warp"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        res.setdefault(d.get("Metric Name"), f"{d.get('Metric Value')} {d.get('Metric Unit')}")
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {n: (v[h.index(n)], u[h.index(n)]) for n in names if n in h}


def sass_hot(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    data = []
    for r in rows[2:]:
        try:
            data.append((r[ix["Source"]], int(r[ix["Instructions Executed"]] or 0),
                         int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
        except (ValueError, IndexError):
            pass
    te = sum(d[1] for d in data) or 1
    ts = sum(d[2] for d in data) or 1
    lines = [f"  {d[2] / ts * 100:5.1f}% stall {d[1] / te * 100:5.2f}% exec  {d[0][:80]}"
             for d in sorted(data, key=lambda x: -x[2])[:top]]
    return lines


if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    for k in KEYS:
        if k in d:
            print(f"{k:40s} {d[k]}")
    for k, (v, u) in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                               "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
                               "gpu__time_duration.sum"]).items():
        print(f"{k:40s} {v} {u}")
    if "--sass" in sys.argv:
        print("top stall sites:")
        print("\n".join(sass_hot(rep)))
