"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size")
tot = collections.defaultdict(float)
cnt = collections.Counter()
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
    name = r[ki].split("(")[0].split("::")[-1] + " " + r[gi]
    tot[name] += v
    cnt[name] += 1
    seq.append((name, v))
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / 1e3:9.3f} ms {cnt[k]:4d} x {v / cnt[k]:9.1f} us  {100 * v / T:5.1f}%  {k}")
print(f"total {T / 1e3:.3f} ms over {sum(cnt.values())} launches")
if len(sys.argv) > 2:
    for n, v in seq:
        print(f"{v:10.1f} {n}")
