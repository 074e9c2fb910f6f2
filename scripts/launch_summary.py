"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into per-kernel totals and
shares of the step: python scripts/launch_summary.py launches.csv "<command>" > summary.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    cnt[name] += 1
all_ms = sum(tot.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) of")
print("  " + (sys.argv[2] if len(sys.argv) > 2 else "?"))
print(f"raw: {sys.argv[1]}\n")
for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{name[:60]:60s} launches={cnt[name]:3d} total_ms={ms:10.3f} share={100 * ms / all_ms:5.1f}%")
