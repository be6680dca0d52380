"""Stall-reason breakdown (warp cycles per issued instruction by reason) and pipe use of an ncu capture."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:60])
    st = []
    for k, v in d.items():
        if "average_warp_latency_issue_stalled" in k or "average_warps_issue_stalled" in k and k.endswith(".ratio"):
            try:
                st.append((float(v), k))
            except ValueError:
                pass
    for v, k in sorted(st, reverse=True)[:12]:
        print(f"  {v:8.3f}  {k}")
    for k, v in d.items():
        if ("pipe" in k and "pct_of_peak_sustained_active" in k) or "throughput.avg.pct_of_peak_sustained_elapsed" in k:
            try:
                if float(v) > 10:
                    print(f"  {float(v):8.2f}  {k}")
            except ValueError:
                pass
