"""Summaries of ncu outputs: launch-list CSV aggregation and per-kernel details."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        agg.setdefault(r[ki].split("(")[0][:48], []).append(float(r[vi].replace(",", "")))
    out = []
    for k, v in agg.items():
        out.append((k, len(v), sum(v) / len(v) / 1000.0))
    return out


WANT = ("Duration", "Executed Ipc Active", "Issue Slots Busy", "DRAM Throughput", "Achieved Occupancy",
        "Executed Instructions", "Registers Per Thread", "Theoretical Occupancy", "L2 Hit Rate", "Grid Size",
        "Memory Throughput", "No Eligible", "Warp Cycles Per Issued Instruction")


def details(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h = r[0]
    cur = None
    lines = []
    for row in r[1:]:
        d = dict(zip(h, row))
        k = d["Kernel Name"][:40] + " #" + d["ID"]
        if k != cur:
            lines.append("== " + k)
            cur = k
        if d["Metric Name"] in WANT:
            lines.append(f"   {d['Metric Name'][:40]:40s} {d['Metric Value']} {d['Metric Unit']}")
    return lines


def raw(rep, metrics):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h = r[0]
    out = []
    for row in r[2:]:
        d = dict(zip(h, row))
        out.append((d["Kernel Name"][:40], {m: d.get(m) for m in metrics}))
    return out


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        for k, n, us in launches(sys.argv[2]):
            print(f"{k:48s} n={n:3d} mean_us={us:8.2f}")
    elif sys.argv[1] == "details":
        print("\n".join(details(sys.argv[2])))
    elif sys.argv[1] == "raw":
        for k, d in raw(sys.argv[2], sys.argv[3].split(",")):
            print(k, d)
