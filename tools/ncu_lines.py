"""Per-CUDA-source-line totals of an ncu capture (warp stall samples and warp instructions
executed), from `ncu -i REP --page source --csv --print-source cuda,sass`.  Dev tool.
  python tools/ncu_lines.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = []
    fname = "?"
    hdr = None
    for r in csv.reader(out):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("Function Name",):
            continue
        try:
            if r[2] != "-":  # sass rows carry an address; cuda rows have "-"
                continue
            samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            exe = int(r[hdr.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((samp, exe, f"{fname}:{r[0]}", r[1].strip()))
    ts = sum(x[0] for x in rows) or 1
    te = sum(x[1] for x in rows) or 1
    print(f"samples {ts}  warp instructions {te}")
    for s, e, loc, src in sorted(rows, reverse=True)[:top]:
        print(f"{100*s/ts:5.1f}% smp {100*e/te:5.1f}% exe  {loc:24s} {src[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
