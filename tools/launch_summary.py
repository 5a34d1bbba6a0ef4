"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel launches / mean / total / share (python tools/launch_summary.py X.csv)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0] != "ID"]
acc = collections.OrderedDict()
for r in rows:
    name = r[4].split("(")[0]
    if r[12] != "gpu__time_duration.sum":
        continue
    v = float(r[14].replace(",", ""))
    us = v / 1e3 if r[13] == "ns" else (v * 1e3 if r[13] == "ms" else v)
    n, t = acc.get(name, (0, 0.0))
    acc[name] = (n + 1, t + us)
tot = sum(t for _, t in acc.values())
print("kernel,launches,mean_us,total_us,share")
for k, (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{k},{n},{t / n:.2f},{t:.1f},{t / tot:.3f}")
