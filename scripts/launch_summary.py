"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per
kernel, share of the summed duration, mean duration and count."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("(anonymous namespace)::", "")[:72]
    tot[k] += float(d["Metric Value"])
    cnt[k] += 1
T = sum(tot.values())
print(f"# {sum(cnt.values())} launches, summed duration {T / 1e3:.1f} us (ncu serialises launches: shares, not wall time)")
for k, v in tot.most_common():
    print(f"{v / T * 100:6.2f}%  {v / cnt[k] / 1e3:9.2f} us  x{cnt[k]:4d}  {k}")
