"""Summarise an ncu report (--set full) or a launch-list CSV into profiles/.

    python scripts/ncu_summary.py report gpurun_out/x.ncu-rep > profiles/x.txt
    python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/x_launches.txt
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    r"^gpu__time_duration\.sum$",
    r"^launch__grid_size$", r"^launch__block_size$", r"^launch__registers_per_thread$",
    r"^sm__pipe_tensor_cycles_active\.avg\.pct_of_peak_sustained_active$",
    r"^sm__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^gpu__compute_memory_throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^dram__bytes_read\.sum$", r"^dram__bytes_write\.sum$",
    r"^gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^lts__t_bytes\.sum$",
    r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"^smsp__sass_inst_executed_op_utcmma\.sum$",
    r"^smsp__pcsamp_warps_issue_stalled_(long_scoreboard|barrier|wait|short_scoreboard|no_instructions|math_pipe_throttle|mio_throttle|lg_throttle)$",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = [i for i, h in enumerate(hdr) if any(re.search(k, h) for k in KEYS)]
    kn = hdr.index("Kernel Name")
    for r in rows[2:]:
        print(f"== {r[kn][:110]}")
        for i in idx:
            if r[i] not in ("", "0"):
                print(f"   {hdr[i]:<75} {r[i]:>16} {units[i]}")


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, gi, bi, mi, ni = (hdr.index(k) for k in ("Kernel Name", "Grid Size", "Block Size", "Metric Value",
                                                 "Metric Name"))
    tot = {}
    n = 0
    print(f"{'us':>10}  grid          block        kernel")
    for r in rows[1:]:
        if len(r) <= mi or r[ni] != "gpu__time_duration.sum":
            continue
        us = float(r[mi]) / 1e3
        name = re.sub(r"\(.*", "", r[ki])[:90]
        print(f"{us:10.2f}  {r[gi]:<13} {r[bi]:<12} {name}")
        tot[name] = tot.get(name, 0.0) + us
        n += 1
    print(f"\n{n} launches; time by kernel (cold, serialised by ncu: compare shares, not absolutes):")
    s = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{v:10.2f} us  {100 * v / s:5.1f}%  {k}")


if __name__ == "__main__":
    {"report": report, "launches": launches}[sys.argv[1]](sys.argv[2])
