"""Summarise an ncu launch list (--metrics gpu__time_duration.sum[,dram__bytes_*] --csv).

usage: python tools/ncu_launches.py launches.csv
Prints per-kernel launch counts, total/avg duration, share of device time and
DRAM bytes per launch (cold-cache, serialised replay: shares, not absolutes).
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
per = collections.defaultdict(dict)
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    per[(int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0])][r[ix["Metric Name"]]] = float(
        r[ix["Metric Value"]].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, name), m in per.items():
    a = agg[name]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s} {'dram_MB/launch':>15s}")
for name, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:40s} {n:8d} {t/1e3:10.1f} {t/n/1e3:9.2f} {100*t/tot:6.1f}% {b/n/1e6:15.2f}")
