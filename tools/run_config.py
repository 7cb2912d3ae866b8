"""Time a few generations of one BASELINE config on the device (graph mode).

    python tools/run_config.py --config c3 [--gens 20] [--warm 5] [--algo hybrid]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CONFIGS = {
    "c1": dict(NP=50, D=1000, G=500, t=1.0, pumps=(1404.0,), variant="single_thg"),
    "c2": dict(NP=1024, D=10_000, G=1000, t=1.0, pumps=(1404.0,), variant="single_thg"),
    "c3": dict(NP=8192, D=100_000, G=1000, t=0.1, pumps=(1404.0,), variant="single_thg"),
    "c4": dict(NP=4096, D=10_000, G=1000, t=1.0, pumps=(1404.0,), variant="single_thg"),
    "c5": dict(NP=2048, D=20_000, G=1000, t=0.5, pumps="linspace", variant="multi_thg"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--gens", type=int, default=20)
    ap.add_argument("--warm", type=int, default=20)  # >= QPM_GRAPH_GENS: the multi-generation graph is built before timing
    ap.add_argument("--algo", default="hybrid")
    ap.add_argument("--profile", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    cfg = CONFIGS[args.config]
    pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, 64)) if cfg["pumps"] == "linspace" else cfg["pumps"]
    spec = q.ObjectiveSpec(cfg["variant"], pumps)
    t0 = time.perf_counter()
    obj = q.make_objective(spec, q.default_dispersion(), cfg["t"], cfg["D"])
    gwo = q.GWOParams(a=0.1, a_final=0.01) if args.algo == "gwo" else q.GWOParams()
    eng = q.Engine(obj, args.algo, pop_size=cfg["NP"], generations=cfg["G"], seed=0, de=q.DEParams(), gwo=gwo,
                   sch=q.Schedules())
    eng.init()
    eng.prepare(args.gens)  # graph replays in the timed window (as bench.py)
    eng.step(args.warm)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    s = eng.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.step(args.gens)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.gens
    stages = eng.profile(args.profile) if args.profile else []
    nwl = len(pumps)
    k = 3 if args.algo == "gwo" else 4
    rows = {"hybrid": 2 * cfg["NP"] - k, "de": cfg["NP"], "gwo": cfg["NP"] - 3}[args.algo]
    evals = rows * cfg["D"] * nwl
    print(json.dumps({"config": args.config, "algo": args.algo, "NP": cfg["NP"], "D": cfg["D"], "n_wl": nwl,
                      "ms_per_gen": ms, "gen_per_s": 1e3 / ms, "domain_evals_per_s": evals / (ms * 1e-3),
                      "setup_s": setup, "device_GB": eng.device_bytes / 1e9, "stages": stages,
                      "best": float(eng.trace()[-1, 1])}))


if __name__ == "__main__":
    main()
