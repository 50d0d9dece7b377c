"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel total time, share and average (shares are what matter: ncu
serialises launches and runs them cold-cache)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0][:90]
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{'total_us':>10} {'share':>6} {'n':>5} {'avg_us':>9}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} {100 * v / T:5.1f}% {cnt[k]:5d} {v / cnt[k]:9.2f}  {k}")
