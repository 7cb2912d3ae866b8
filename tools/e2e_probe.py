"""Where the end-to-end seconds of a short public run_hybrid call go (C2 shape).

    python tools/e2e_probe.py [--gens 20] [--reps 5]

Prints, per repetition, the host-timed phases of an Engine driven by hand
(create, init, graph capture, generations, finalize, read-back, destroy), the
same run with eager launches instead of graphs, and the public run_hybrid()
call, as JSON lines.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200.optimizer import DEParams, Engine, GWOParams, Schedules

    torch.cuda.set_device(0)
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 10_000)
    G = args.gens
    for rep in range(args.reps):
        for mode in ("graph", "eager"):
            marks = []
            t0 = time.perf_counter()

            def mark(name):
                torch.cuda.synchronize()
                marks.append((name, time.perf_counter()))

            eng = Engine(obj, "hybrid", pop_size=1024, generations=G, seed=0, de=DEParams(), gwo=GWOParams(),
                         sch=Schedules())
            mark("create")
            eng.init()
            mark("init")
            if mode == "graph":
                eng.prepare(G)
                mark("capture")
            eng.step(G, use_graph=mode == "graph")
            mark("steps")
            eng.finalize()
            eng.trace(0, G + 1)
            eng.best()
            mark("finalize_read")
            del eng
            mark("destroy")
            prev, parts = t0, {}
            for n, tt in marks:
                parts[n] = round(1e3 * (tt - prev), 3)
                prev = tt
            print(json.dumps({"rep": rep, "mode": mode, "total_ms": round(1e3 * (prev - t0), 3), **parts}))
        t1 = time.perf_counter()
        q.run_hybrid(obj, dimension=10_000, pop_size=1024, generations=G, seed=0)
        torch.cuda.synchronize()
        print(json.dumps({"rep": rep, "mode": "run_hybrid", "total_ms": round(1e3 * (time.perf_counter() - t1), 3)}))


if __name__ == "__main__":
    main()
