"""Per-kernel achieved DRAM bandwidth from an ncu CSV with gpu__time_duration.sum,
dram__bytes_read.sum and dram__bytes_write.sum (one low-rank config-2 step;
ncu flushes the caches before each replay, so these are cold-cache figures)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
per = collections.defaultdict(lambda: collections.defaultdict(float))
unit = {}
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    k = (d["ID"], re.sub(r"\(.*", "", d["Kernel Name"]).replace("(anonymous namespace)::", "")[:70])
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "msecond": 1e-3, "nsecond": 1e-9}.get(u, 1)
    per[k][d["Metric Name"]] = v * scale
kinds = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, name), m in per.items():
    t = m.get("gpu__time_duration.sum", 0)
    b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a = kinds[name]
    a[0] += 1
    a[1] += t
    a[2] += b
print("# kernel, launches, mean us, mean DRAM MB, achieved GB/s (cold cache, ncu-serialised)")
for name, (c, t, b) in sorted(kinds.items(), key=lambda x: -x[1][1]):
    print(f"{c:4d}  {t / c * 1e6:9.2f} us  {b / c / 1e6:9.3f} MB  {b / t / 1e9 if t else 0:8.0f} GB/s  {name}")
