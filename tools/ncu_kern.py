"""Per-kernel key counters of an ncu capture (duration, DRAM bytes, instructions, issue).  Dev tool."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:45], " ".join(f"{k.split('.')[0].split('__')[1]}={d.get(k, '?')}" for k in keys))
