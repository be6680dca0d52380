"""Launch list (ncu --metrics gpu__time_duration.sum --csv) -> markdown table per kernel.
    python tools/launches_md.py launches.csv "<title>" > launches.md"""
import csv
import statistics
import sys
from collections import OrderedDict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
per = OrderedDict()
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    u = r[iu]
    us = v / 1e3 if u in ("ns", "nsecond") else (v * 1e3 if u in ("ms", "msecond") else v)
    per.setdefault(r[ik], []).append(us)
print(f"# {sys.argv[2]}\n")
print("`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` (tools/gpu_final_r2.sh).")
print("Per-launch times under ncu are cold-cache and serialised: compare shares, not absolutes.")
print("Several launches of one kernel include the e2e legs (chunked launches over pinned host")
print("buffers) and the warm-up; the full-size step launches are the maxima.\n")
print("| launches | min µs | median µs | max µs | kernel |\n|---|---|---|---|---|")
for k, v in per.items():
    name = k.split("(")[0][:90]
    print(f"| {len(v)} | {min(v):.1f} | {statistics.median(v):.1f} | {max(v):.1f} | `{name}` |")
