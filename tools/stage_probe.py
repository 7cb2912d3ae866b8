"""Per-stage device time of one engine generation (Engine.profile: CUDA events between stages, eager).

    python tools/stage_probe.py NP D [NP D ...]  [--warm 30] [--gens 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("shape", nargs="+", type=int)
    ap.add_argument("--warm", type=int, default=30)
    ap.add_argument("--gens", type=int, default=20)
    args = ap.parse_args()
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    for NP, D in zip(args.shape[::2], args.shape[1::2]):
        obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, D)
        eng = q.Engine(obj, "hybrid", pop_size=NP, generations=1000, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                       sch=q.Schedules())
        eng.init()
        eng.step(args.warm)
        st = eng.profile(args.gens)
        print(json.dumps({"NP": NP, "D": D, "total_us": round(1e3 * sum(m for _, m in st), 1),
                          "stages_us": {n: round(1e3 * m, 1) for n, m in st}}), flush=True)
        del eng


if __name__ == "__main__":
    main()
