"""Summarise an ncu --page source capture: hottest SASS lines by stall samples and
instruction execution counts (reads `ncu -i <rep> --page source --csv`)."""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    while rows and "Address" not in rows[0]:
        rows = rows[1:]
    h = rows[0]
    ia, isrc, isamp, iexe = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    data = []
    for r in rows[1:]:
        try:
            data.append((int(r[isamp] or 0), int(r[iexe] or 0), r[ia], r[isrc].strip()))
        except (ValueError, IndexError):
            pass
    tot_s = sum(d[0] for d in data)
    tot_e = sum(d[1] for d in data)
    print(f"total samples {tot_s}, warp instructions executed {tot_e}")
    for s, e, a, src in sorted(data, reverse=True)[:top]:
        print(f"{s:7d} {100*s/max(tot_s,1):5.1f}%  exe {e:10d}  {src[:90]}")
    # executed-instruction histogram by opcode
    from collections import Counter
    c = Counter()
    for s, e, a, src in data:
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        c[op.split(".")[0]] += e
    print("executed by opcode:", ", ".join(f"{k}:{v/tot_e*100:.1f}%" for k, v in c.most_common(18)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
