"""Host-side cost of each call of a short public run (C2 shape, K generations).

    python tools/e2e_detail.py [--gens 20] [--reps 8]

Every phase is bracketed by torch.cuda.synchronize() and timed on the host
clock; the median over reps is printed as one JSON line per phase.
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=20)
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200 import _native
    from paper_2511_01255_b200.optimizer import DEParams, Engine, GWOParams, Schedules, _trace_rows, schedule_table

    torch.cuda.set_device(0)
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 10_000)
    G, NP = args.gens, 1024
    de, gwo, sch = DEParams(), GWOParams(), Schedules()
    times = {}

    def t(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        times.setdefault(name, []).append(1e3 * (time.perf_counter() - t0))
        return r

    for rep in range(args.reps + 2):
        t("schedule_table", lambda: schedule_table(G, de, gwo, sch))
        eng = t("Engine()", lambda: Engine(obj, "hybrid", pop_size=NP, generations=G, seed=rep, de=de, gwo=gwo,
                                           sch=sch))
        t("init", eng.init)
        t("step(eager)", lambda: eng.step(G))
        t("finalize", eng.finalize)
        tr = t("trace", lambda: eng.trace(0, G + 1))
        t("trace_rows", lambda: _trace_rows(tr))
        t("best", eng.best)
        t("del", lambda: eng.__del__())
        t("run_hybrid", lambda: q.run_hybrid(obj, dimension=10_000, pop_size=NP, generations=G, seed=rep))
    for k, v in times.items():
        print(json.dumps({"phase": k, "median_ms": float(np.median(v[2:])), "min_ms": float(np.min(v[2:]))}))


if __name__ == "__main__":
    main()
