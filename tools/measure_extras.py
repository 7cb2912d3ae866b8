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
