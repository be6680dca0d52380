"""Summarise ncu captures into profiles/: a markdown table of the key counters per kernel,
the per-kernel DRAM traffic (profiles/traffic.json, read by bench.py for roofline.traffic)
and the launch list shares.

    python tools/profile_summary.py <round-tag> <launches.csv> <rep1.ncu-rep> [<rep2> ...]
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def raw(rep):
    """rep: an .ncu-rep, or the `ncu -i <rep> --page raw --csv` export of one (*.csv)"""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({name: (r[i], units[i]) for i, name in enumerate(h)})
    return res


def main():
    tag, launches, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary ({tag})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 (gpurun), "
             "one launch per kernel after warm-up.  Raw reports stay in gpurun_out/ (scratch); this file and "
             "traffic.json are the committed evidence.", ""]
    traffic = {}
    for rep in reps:
        for k in raw(rep):
            name = k.get("Kernel Name", ("?", ""))[0]
            short = name.split("(")[0].replace("void ", "").replace("br::", "")
            lines.append(f"## {short}  ({os.path.basename(rep)})")
            lines.append("")
            lines.append("| counter | value |")
            lines.append("|---|---|")
            for m, label in METRICS:
                if m in k:
                    v, u = k[m]
                    lines.append(f"| {label} (`{m}`) | {v} {u} |")
            if "dram__bytes_read.sum" in k and "dram__bytes_write.sum" in k:
                t = to_bytes(*k["dram__bytes_read.sum"]) + to_bytes(*k["dram__bytes_write.sum"])
                traffic[short.split("<")[0]] = t
                lines.append(f"| dram read+write per launch | {t/1e6:.1f} MB |")
            lines.append("")
    # launch list shares
    if launches and os.path.exists(launches):
        rows = list(csv.reader(open(launches)))
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        agg = defaultdict(list)
        for r in rows[hdr + 1:]:
            if len(r) > vi:
                v = float(r[vi].replace(",", ""))
                v *= {"ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}.get(r[ui], 1)
                agg[r[ki].split("(")[0].replace("void ", "")].append(v)
        tot = sum(sum(v) for v in agg.values())
        lines += ["## launch list (gpu__time_duration.sum, cold-cache, serialised)", "",
                  "| kernel | launches | mean us | share of captured time |", "|---|---|---|---|"]
        for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {name[:80]} | {len(v)} | {sum(v)/len(v):.1f} | {100*sum(v)/tot:.1f}% |")
        lines.append("")
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as fh:
        fh.write("\n".join(lines))
    old = {}
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        old = json.load(open(tp))
    old.update(traffic)
    json.dump(old, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
