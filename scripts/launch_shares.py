"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel time shares.  usage: launch_shares.py launches.csv [title]"""
import csv
import collections
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    if len(r) <= vi or r[ki] == "Kernel Name":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
    name = r[ki]
    if "nvjet" in name or "gemm" in name.lower():
        name = "cuBLASLt GEMM " + name.split("(")[0][:60]
    else:
        name = name.split("(")[0]
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"total {T:.0f} ms over {sum(cnt.values())} launches")
for n, t in tot.most_common(25):
    print(f"{100 * t / T:6.2f}% {t:10.1f} ms {cnt[n]:5d} launches  {n}")
