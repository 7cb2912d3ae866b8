"""Time C2 generations (graph replay) for several engine settings in one process.

    python tools/gen_sweep.py 'QPM_PDL=0' 'QPM_PDL=1' 'QPM_WOLF=planner,QPM_PLAN_FORK=trial,QPM_PLAN_CTAS=296'
Each argument is a comma-separated env assignment list applied before the engine is created
(QPM_SWEEP_SHAPE="NP,D" and QPM_SWEEP_ALGO=hybrid|de|gwo in the environment change the run from C2 hybrid)
(the QPM_* knobs are read at engine / problem creation).  Every setting times the same
generations (warm-up 50, then 3 x 300), reported as the median us per generation.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    os.environ.setdefault("QPM_DEV_KNOBS", "1")  # scheduling knobs are read only with this set
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    configs = sys.argv[1:] or [""]
    keys = set()
    for cfg in configs:
        for kv in filter(None, cfg.split(",")):
            keys.add(kv.split("=")[0])
    for cfg in configs:
        for k in keys:
            os.environ.pop(k, None)
        for kv in filter(None, cfg.split(",")):
            k, v = kv.split("=")
            os.environ[k] = v
        NPs, Ds = (int(x) for x in os.environ.get("QPM_SWEEP_SHAPE", "1024,10000").split(","))
        obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, Ds)
        algo = os.environ.get("QPM_SWEEP_ALGO", "hybrid")
        gwo = q.GWOParams(a=0.1, a_final=0.01) if algo == "gwo" else q.GWOParams()
        eng = q.Engine(obj, algo, pop_size=NPs, generations=1000, seed=0, de=q.DEParams(), gwo=gwo,
                       sch=q.Schedules())
        eng.init()
        eng.step(50)
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
            eng.step(300)
            e1.record(eng.stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3 / 300)
        print(f"{cfg or 'default':70s} {np.median(times):8.2f} us/gen  {['%.1f' % t for t in times]}"
              f"  best={eng.trace()[-1][1]:.6g}", flush=True)
        del eng


if __name__ == "__main__":
    main()
