"""Per-kernel achieved DRAM bandwidth from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(serialised, cold-cache launches): `python tools/hbm_table.py launches.csv [peak_GBps]`."""
import csv
import sys
from collections import defaultdict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
        "second": 1.0}


def main():
    path = sys.argv[1]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else None
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    per = defaultdict(dict)
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        per[key][r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in per.items():
        a = agg[name[:70]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    print(f"{'total_ms':>9} {'share':>6} {'n':>4} {'avg_us':>9} {'MB/launch':>10} {'GB/s':>7} {'%peak':>6}  kernel")
    for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        bw = b / t / 1e9 if t else 0.0
        pk = f"{100 * bw / peak:6.1f}" if peak else "     -"
        print(f"{t * 1e3:9.3f} {100 * t / total:5.1f}% {n:4d} {t / n * 1e6:9.1f} {b / n / 1e6:10.1f} {bw:7.0f} {pk}  {name}")


if __name__ == "__main__":
    main()
