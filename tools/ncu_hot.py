"""Top stall-sampled SASS lines of one kernel in an ncu report.

    python tools/ncu_hot.py REPORT KERNEL_REGEX [N]
"""
import csv
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre,
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h = r[1]
    rows = [dict(zip(h, x)) for x in r[2:] if len(x) == len(h) and x[0] != 'Address']
    si = "Warp Stall Sampling (All Samples)"
    tot = sum(float(x[si] or 0) for x in rows)
    stall_cols = [c for c in h if c.startswith("stall_")]
    print(f"{len(rows)} sass lines, {tot:.0f} samples")
    agg = {c: sum(float(x[c] or 0) for x in rows) for c in stall_cols}
    print("stalls:", ", ".join(f"{k[6:]}={v / tot:.0%}" for k, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
    for i, x in sorted(enumerate(rows), key=lambda t: -float(t[1][si] or 0))[:n]:
        top = sorted(((float(x[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"{i:5d} {float(x[si] or 0) / tot:6.1%} {x['Source'].strip()[:60]:60s} {top}")


if __name__ == "__main__":
    main()
