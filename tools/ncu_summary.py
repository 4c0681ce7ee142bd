"""Summarise ncu output for profiles/ (tracked).

  python tools/ncu_summary.py launches <launches.csv>       per-kernel share of one step
  python tools/ncu_summary.py report <file.ncu-rep>         key counters of a --set full capture

Prints markdown; the caller redirects it under profiles/.
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "SM Frequency"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Scheduler Statistics", "No Eligible"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Occupancy", "Achieved Occupancy"),
]
RAW = [
    r"^dram__bytes_read\.sum$", r"^dram__bytes_write\.sum$", r"^gpu__time_duration\.sum$",
    r"^sm__inst_executed_pipe_(xu|fma|alu|lsu|fp64)\.avg\.pct_of_peak_sustained_active$",
    r"^sm__pipe_(fma|alu|fp64|shared)_cycles_active\.avg\.pct_of_peak_sustained_active$",
    r"^l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum$",
    r"^l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum$",
    r"^l1tex__throughput\.avg\.pct_of_peak_sustained_active$",
    r"^smsp__inst_executed\.sum$",
    r"^smsp__average_warps_issue_stalled_(long_scoreboard|short_scoreboard|wait|mio_throttle|"
    r"math_pipe_throttle|barrier|lg_throttle|not_selected)_per_issue_active\.ratio$",
]


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args + ["--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path):
    rows = ncu_csv(["-i", path, "--page", "details"])
    h = rows[0]
    kn, si, mi, ui, vi = (h.index(x) for x in
                          ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    print(f"### {path.split('/')[-1]}: `{rows[1][kn][:90]}`\n")
    print("| section | metric | value |\n|---|---|---|")
    for r in rows[1:]:
        if (r[si], r[mi]) in KEYS:
            print(f"| {r[si]} | {r[mi]} | {r[vi]} {r[ui]} |")
    raw = ncu_csv(["-i", path, "--page", "raw"])
    h, u, v = raw[0], raw[1], raw[2]
    print("\n| raw counter | value |\n|---|---|")
    for i, n in enumerate(h):
        if any(re.search(p, n) for p in RAW):
            print(f"| {n} | {v[i]} {u[i]} |")
    print()


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > vi and r[vi]:
            n = re.split(r"[(<]", r[ki].replace("void ", ""))[0].strip()
            agg[n][0] += 1
            agg[n][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"### launch list `{path.split('/')[-1]}` (gpu__time_duration.sum, cold, serialised)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {v[0]} | {v[1] / 1e6:.3f} | {v[1] / tot * 100:.1f}% |")
    print(f"| **total** | {sum(v[0] for v in agg.values())} | {tot / 1e6:.3f} | |\n")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
