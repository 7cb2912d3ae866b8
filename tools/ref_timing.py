"""Truncated C2 timing of the reference package itself (qpmdesign, numba backend)
on this host's cores -- context for the CPU baseline, not the reference arm.

    python tools/ref_timing.py [--gens 2]

Imports qpmdesign from baseline/_ref (the pip install of /root/reference/pkg,
DESIGN.md §4), JIT-warms its numba kernels on a tiny problem, then times
run_hybrid at the C2 shape (NP 1024, D 10^4, THG 1404 nm, t 1 um) with
workers = os.cpu_count() for G = 1 and G = 1 + gens; the difference / gens is
the per-generation time (init and generation-0 evaluation excluded, as in
SURVEY.md §8(d)).  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gens", type=int, default=2)
    args = ap.parse_args()
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "qpmdesign")):
        print(json.dumps({"unavailable": "baseline/_ref/qpmdesign is not installed"}))
        return
    sys.path.insert(0, ref)
    import numpy as np
    from qpmdesign import _kernels, optimizer
    from qpmdesign.objectives import ObjectiveSpec, make_objective
    from qpmdesign.physics import default_dispersion

    workers = os.cpu_count() or 1
    spec = ObjectiveSpec("single_thg", (1404.0,))
    t0 = time.perf_counter()
    small = make_objective(spec, default_dispersion(25.0), 1.0, 64)
    optimizer.run_hybrid(small, dimension=64, pop_size=8, generations=2, seed=0, workers=2)
    jit_s = time.perf_counter() - t0
    obj = make_objective(spec, default_dispersion(25.0), 1.0, 10_000)
    times = {}
    for G in (1, 1 + args.gens):
        t0 = time.perf_counter()
        optimizer.run_hybrid(obj, dimension=10_000, pop_size=1024, generations=G, seed=0, workers=workers)
        times[G] = time.perf_counter() - t0
    per_gen = (times[1 + args.gens] - times[1]) / args.gens
    evals = (2 * 1024 - 4) * 10_000
    print(json.dumps({"value": evals / per_gen, "unit": "domain-evals/s", "s_per_generation": per_gen,
                      "cores": workers, "backend": _kernels.backend(), "jit_warmup_s": jit_s,
                      "sample": f"qpmdesign.optimizer.run_hybrid (baseline/_ref) C2 shape, generations 2..{1 + args.gens} "
                                f"(G=1 and G={1 + args.gens} runs differenced), workers={workers}",
                      "numpy": np.__version__}))


if __name__ == "__main__":
    main()
