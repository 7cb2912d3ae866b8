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


# (scale applies after conversion to ns / bytes)
TABLE = [("us", "gpu__time_duration.sum", 1e-3), ("DRAM_rd_MB", "dram__bytes_read.sum", 1e-6),
         ("DRAM_wr_MB", "dram__bytes_write.sum", 1e-6), ("Minst", "smsp__inst_executed.sum", 1e-6),
         ("ALU%", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
         ("FMAheavy%", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
         ("FP64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
         ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
         ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
         ("smem%", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
         ("regs", "launch__registers_per_thread", 1), ("grid", "launch__grid_size", 1)]


def table(rep):
    """One line per captured kernel: duration, DRAM traffic, instructions, pipe use (raw page)."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units = r[0], r[1]
    out = [f"{'kernel':34s} " + " ".join(f"{n:>10s}" for n, _, _ in TABLE)]
    for row in r[2:]:
        d = dict(zip(h, row))
        vals = []
        for n, m, sc in TABLE:
            v = d.get(m, "")
            try:
                x = float(v.replace(",", ""))
                u = units[h.index(m)] if m in h else ""
                if m.startswith("dram__bytes"):  # ncu may report KB/MB/GB
                    x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
                          "GB": 1e9}.get(u, 1)
                if m == "gpu__time_duration.sum":
                    x *= {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(u, 1)
                vals.append(f"{x * sc:10.2f}")
            except ValueError:
                vals.append(f"{'-':>10s}")
        out.append(f"{d['Kernel Name'].split('(')[0][:34]:34s} " + " ".join(vals))
    return out


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        for k, n, us in launches(sys.argv[2]):
            print(f"{k:48s} n={n:3d} mean_us={us:8.2f}")
    elif sys.argv[1] == "details":
        print("\n".join(details(sys.argv[2])))
    elif sys.argv[1] == "table":
        print("\n".join(table(sys.argv[2])))
    elif sys.argv[1] == "raw":
        for k, d in raw(sys.argv[2], sys.argv[3].split(",")):
            print(k, d)
