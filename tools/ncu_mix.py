"""Dynamic SASS instruction mix (and per-unit counts) of one kernel in an ncu report.

    python tools/ncu_mix.py REPORT KERNEL_REGEX [UNITS]
UNITS (e.g. genes per launch) turns warp-instruction counts into thread instructions per unit.
"""
import collections
import csv
import re
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    units = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h = r[1]
    rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h) and x[0] != "Address"]
    half = len(rows) // 2
    if half and rows[0]["Address"] == rows[half]["Address"]:
        rows = rows[:half]
    agg = collections.Counter()
    tot = 0.0
    for x in rows:
        n = float(x["Instructions Executed"] or 0)
        s = re.sub(r"^@!?U?P\w+\s+", "", x["Source"].strip())
        op = s.split()[0] if s else "?"
        base = op.split(".")[0]
        key = op if base == "IMAD" and any(t in op for t in ("WIDE", "HI", "MOV", "IADD", "SHL", "X")) else base
        agg[key] += n
        tot += n
    print(f"total warp instructions {tot:.0f}")
    for k, v in agg.most_common(40):
        per = f"  {v * 32 / units:7.2f} per unit" if units else ""
        print(f"{k:24s} {v / 1e6:8.3f}M {v / tot:6.1%}{per}")


if __name__ == "__main__":
    main()
