"""A C2-shape run for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py [--gens 30] [--np 1024] [--d 10000]
        [--algo hybrid] [--eager] [--env QPM_WOLF=planner,QPM_PLAN_FORK=start]

Runs init + `gens` generations (graph replays with PDL and the side-stream
planner unless --eager), then the finalize / read-back path, and prints a
digest of the trace so runs under the tools can be compared with plain runs.
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    os.environ.setdefault("QPM_DEV_KNOBS", "1")  # scheduling knobs are read only with this set
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=30)
    ap.add_argument("--np", type=int, default=1024)
    ap.add_argument("--d", type=int, default=10_000)
    ap.add_argument("--algo", default="hybrid")
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--env", default="")
    ap.add_argument("--nwl", type=int, default=1)
    args = ap.parse_args()
    for kv in filter(None, args.env.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, args.nwl)) if args.nwl > 1 else (1404.0,)
    spec = q.ObjectiveSpec("multi_thg" if args.nwl > 1 else "single_thg", pumps)
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, args.d)
    gwo = q.GWOParams(a=0.1, a_final=0.01) if args.algo == "gwo" else q.GWOParams()
    eng = q.Engine(obj, args.algo, pop_size=args.np, generations=1000, seed=0, de=q.DEParams(), gwo=gwo,
                   sch=q.Schedules())
    eng.init()
    if not args.eager:
        eng.prepare(args.gens)
    eng.step(args.gens, use_graph=not args.eager)
    eng.finalize()
    t = eng.trace(0, args.gens + 1)
    b = eng.best()
    signs = np.where(np.random.default_rng(0).random((64, args.d)) < 0.5, -1, 1).astype(np.int8)
    f = obj.evaluate_block(signs)
    print("trace", hashlib.sha1(t.tobytes()).hexdigest()[:16], "best", b.fitness, "fit", float(f.sum()), flush=True)


if __name__ == "__main__":
    main()
