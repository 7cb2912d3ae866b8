"""Throughput of the §8(f) extras on one GPU: exhaustive search and batched trials.

    python tools/measure_extras.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    disp = q.default_dispersion()
    for n in (20, 24, 28):
        for mode in ("exact", "fast"):
            obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, n, mode=mode)
            t0 = time.perf_counter()
            signs, fit = q.brute_force_oracle(obj, n, limit=64, chunk=1 << 22)
            dt = time.perf_counter() - t0
            print(f"brute_force n={n} mode={mode}: {dt * 1e3:9.1f} ms, {(1 << n) / dt:.3e} patterns/s, "
                  f"{(1 << n) * n / dt:.3e} domain-evals/s, best={fit!r}", flush=True)
    # batched spectra: 64 patterns x 1000 wavelengths at D = 2e4 (C5's wavelength axis)
    import numpy as np

    rng = np.random.default_rng(0)
    signs = np.where(rng.random((64, 20_000)) < 0.5, -1, 1).astype(np.int8)
    wls = np.linspace(1300.0, 1650.0, 1000)
    q.sweep_spectra(signs[:2], 0.5, disp, wls[:10], "thg")
    for process in ("thg", "shg"):
        t0 = time.perf_counter()
        out = q.sweep_spectra(signs, 0.5, disp, wls, process)
        dt = time.perf_counter() - t0
        print(f"sweep_spectra {process} 64 patterns x 1000 wl x D 2e4: {dt * 1e3:.1f} ms "
              f"({out.size * 20_000 / dt:.3e} domain-evals/s incl. host dispersion + transfers)", flush=True)
    # C1 trials: NP 50, D 1000, G 500, 30 seeds (the paper's Tables 3-7 protocol)
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, 1000)
    for algo in ("hybrid", "de", "gwo"):
        q.run_trials(obj, algo, 2, 0, dimension=1000, pop_size=50, generations=20)  # warm
        t0 = time.perf_counter()
        stats, recs = q.run_trials(obj, algo, 30, 0, dimension=1000, pop_size=50, generations=500)
        dt = time.perf_counter() - t0
        print(f"run_trials C1 {algo} x30: {dt:.3f} s total, {dt / 30 * 1e3:.1f} ms per trial, "
              f"mean best {stats.average:.6f} (std {stats.std:.2e})", flush=True)


if __name__ == "__main__":
    main()
