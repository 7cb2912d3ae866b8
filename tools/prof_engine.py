"""Run a few C2 generations eagerly (no graph) for ncu captures.

    python tools/prof_engine.py [--gens N] [--warm W] [--np NP] [--d D] [--algo hybrid]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=2)
    ap.add_argument("--warm", type=int, default=20)
    ap.add_argument("--np", type=int, default=1024)
    ap.add_argument("--d", type=int, default=10_000)
    ap.add_argument("--algo", default="hybrid")
    ap.add_argument("--mode", default="fast")
    args = ap.parse_args()
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, args.d,
                           mode=args.mode)
    eng = q.Engine(obj, args.algo, pop_size=args.np, generations=1000, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                   sch=q.Schedules())
    eng.init()
    eng.step(args.warm, use_graph=True)
    torch.cuda.synchronize()
    eng.step(args.gens, use_graph=False)
    torch.cuda.synchronize()
    print("done", eng.trace()[-1].tolist())


if __name__ == "__main__":
    main()
