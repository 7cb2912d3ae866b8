"""In-graph kernel timeline of C2 generations from a -DQPM_TRACE build.

    python tools/timeline.py [LIB] [--gens N] [--np NP] [--d D] [--algo hybrid]
Builds: python tools/ab_build.py trace='-DQPM_TRACE'  (-> build/ab/libqpm_trace.so).
Prints, per kernel, the mean over generations of: entry (CTA resident, before the
PDL wait), start (after the wait) and end, relative to the generation's first
de_trial start, plus the mean busy time (end - start).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = ["de_trial", "fit_fast", "fit_finish", "topk|fs<0>", "gwo_apply", "stats|fs<1>", "plan_rows", "plan_bump",
         "plan_wolf"]  # ids 3 / 5: k_select_topk / k_select_stats or the fused k_finish_select<0> / <1>
IDS, LEN = 9, 4096


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib", nargs="?", default=os.path.join(ROOT, "build", "ab", "libqpm_trace.so"))
    ap.add_argument("--gens", type=int, default=200)
    ap.add_argument("--warm", type=int, default=600)
    ap.add_argument("--np", type=int, default=1024)
    ap.add_argument("--d", type=int, default=10_000)
    ap.add_argument("--algo", default="hybrid")
    args = ap.parse_args()
    os.environ["QPM_LIB"] = args.lib
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200 import _native

    torch.cuda.set_device(0)
    L = _native.lib()
    fns = [getattr(L, "qpm_dev_trace_engine"), getattr(L, "qpm_dev_trace_fitness")]
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, args.d)
    eng = q.Engine(obj, args.algo, pop_size=args.np, generations=args.warm + args.gens + 10, seed=0,
                   de=q.DEParams(), gwo=q.GWOParams(), sch=q.Schedules())
    eng.init()
    eng.prepare(max(args.gens, 10))  # graph replays from the first generation (as in bench.py)
    eng.prepare(1)
    eng.step(args.warm)
    torch.cuda.synchronize()
    for f in fns:
        assert f(1, None, None) == 0, "not a -DQPM_TRACE build"
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(eng.stream)
    eng.step(args.gens)
    e1.record(eng.stream)
    torch.cuda.synchronize()
    logs, counts = [], []
    for f in fns:
        log = np.zeros((IDS, LEN, 3), dtype=np.uint64)
        cnt = np.zeros(IDS, dtype=np.uint32)
        assert f(0, log.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p)) == 0
        logs.append(log)
        counts.append(cnt)
    # kernel id -> (launch log, count); fitness kernels live in the second unit
    rec = {}
    for k in range(IDS):
        u = 1 if k in (1, 2) else 0
        lg = logs[u][k][:counts[u][k]].copy()
        lg[:, 1] = np.where(lg[:, 1] == np.uint64(2**64 - 1), lg[:, 0], lg[:, 1])  # no QTRACE_STARTED: entry
        rec[k] = (lg.astype(np.int64), int(counts[u][k]))
    g = args.gens
    base = rec[0][0][:, 1]  # de_trial start per generation
    n_per = {k: rec[k][1] // g for k in rec}
    print(f"{g} generations, {e0.elapsed_time(e1) * 1e3 / g:.2f} us/gen (events); launches per gen:",
          {NAMES[k]: n_per[k] for k in rec})
    gen_len = np.diff(base).mean() / 1e3
    print(f"mean generation (de_trial start to start): {gen_len:.2f} us")
    print(f"{'kernel':14s} {'#':>2s} {'entry':>8s} {'start':>8s} {'end':>8s} {'busy':>8s}   (us from de_trial start)")
    rows = []
    for k in range(IDS):
        log, n = rec[k]
        per = n_per[k]
        if per == 0:
            continue
        for r in range(per):
            sel = log[r::per][:g]
            m = min(len(sel), len(base))
            rel = (sel[:m] - base[:m, None]) / 1e3
            rows.append((np.mean(rel[:, 1]), NAMES[k], r, rel))
    for _, name, r, rel in sorted(rows):
        print(f"{name:14s} {r:2d} {rel[:, 0].mean():8.2f} {rel[:, 1].mean():8.2f} {rel[:, 2].mean():8.2f} "
              f"{(rel[:, 2] - rel[:, 1]).mean():8.2f}")
    print("fit_fast CTA 0 stamps (us from start): bits, first table, loop end, stored =",
          [round(float(x), 2) for x in stamps(L)[1:5]])
    print("de_trial CTA 0 stamps (us from start): setup done, thread 0 done =",
          [round(float(x), 2) for x in stamps(L, "qpm_dev_trace_engine", 0)[1:3]])
    for kid in (3, 5):
        print(f"{NAMES[kid]} stamps (us from CTA 0 start): CTA 0 rows done, last CTA detected, last CTA done =",
              [round(float(x), 2) for x in stamps(L, "qpm_dev_trace_engine", kid)[1:4]])
    print("stats|fs<1> last-CTA stamps: state staged, selection + max done, mean done, var done =",
          [round(float(x), 2) for x in stamps(L, "qpm_dev_trace_engine", 5)[4:8]])




def stamps(L, fn_name="qpm_dev_trace_fitness", kid=1, n=8):
    """Intra-kernel stamps of CTA 0 (QSTAMP slots) for kernel id kid, relative to slot 0, in us."""
    import numpy as np

    buf = np.zeros((IDS, 64, 8), dtype=np.uint64)
    assert getattr(L, fn_name)(2, buf.ctypes.data_as(ctypes.c_void_p), None) == 0
    s = buf[kid].astype(np.int64)
    s = s[s[:, 0] > 0]
    if len(s) == 0:
        return np.zeros(n)
    rel = (s[:, :n] - s[:, :1]) / 1e3
    return rel.mean(axis=0)


if __name__ == "__main__":
    main()
