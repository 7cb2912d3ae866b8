"""Runs engine configurations with the library named by QPM_LIB and prints, per
run, the trace digest and (checks build) the invariant-violation flags.
Launched by tests/test_gpu_checks.py; not a test module."""

import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

RUNS = [
    dict(algo="hybrid", NP=1024, D=10_000, G=60, env={}),
    dict(algo="hybrid", NP=96, D=3000, G=40, env={"QPM_WOLF": "planner", "QPM_PLAN_FORK": "start"}),
    dict(algo="hybrid", NP=96, D=3000, G=40, env={"QPM_WOLF": "side"}),
    dict(algo="hybrid", NP=64, D=700, G=30, env={}, leaders=3),
    dict(algo="de", NP=512, D=5000, G=30, env={}),
    dict(algo="gwo", NP=512, D=5000, G=30, env={}),
    dict(algo="hybrid", NP=4200, D=1300, G=8, env={}),
    dict(algo="hybrid", NP=128, D=4000, G=12, env={}, nwl=3),
]


def main():
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200 import _native

    torch.cuda.set_device(0)
    os.environ["QPM_DEV_KNOBS"] = "1"  # the runs below pick scheduling knobs
    out = []
    for k, r in enumerate(RUNS):
        for key in ("QPM_WOLF", "QPM_PLAN_FORK"):
            os.environ.pop(key, None)
        os.environ.update(r["env"])
        nwl = r.get("nwl", 1)
        pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, nwl)) if nwl > 1 else (1404.0,)
        spec = q.ObjectiveSpec("multi_thg" if nwl > 1 else "single_thg", pumps)
        obj = q.make_objective(spec, q.default_dispersion(), 1.0, r["D"])
        gwo = q.GWOParams(a=0.1, a_final=0.01) if r["algo"] == "gwo" else q.GWOParams(
            leader_count=r.get("leaders", 4))
        eng = q.Engine(obj, r["algo"], pop_size=r["NP"], generations=r["G"], seed=k, de=q.DEParams(), gwo=gwo,
                       sch=q.Schedules())
        eng.init()
        eng.prepare(r["G"])
        eng.step(r["G"])
        eng.finalize()
        t = eng.trace()
        flags, detail = np.zeros(1, np.uint32), np.zeros(1, np.uint32)
        rc = _native.lib().qpm_engine_check_status(eng.handle, flags.ctypes.data, detail.ctypes.data)
        out.append({"run": k, "digest": hashlib.sha1(t.tobytes()).hexdigest(), "checks": rc == 0,
                    "flags": int(flags[0]), "detail": int(detail[0])})
        del eng
    print(json.dumps(out))


if __name__ == "__main__":
    main()
