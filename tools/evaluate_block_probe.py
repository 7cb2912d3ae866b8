"""Plug point 1 timing: GpuPatternObjective.evaluate_block on host int8 rows
(the call the reference's own run_hybrid makes through parexec.evaluate_batch).

    python tools/evaluate_block_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q

    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    for tag, rows, d, nwl in (("C2", 2044, 10_000, 1), ("C5", 4092, 20_000, 64)):
        pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, nwl)) if nwl > 1 else (1404.0,)
        spec = q.ObjectiveSpec("multi_thg" if nwl > 1 else "single_thg", pumps)
        obj = q.make_objective(spec, q.default_dispersion(), 0.5 if nwl > 1 else 1.0, d)
        signs = np.where(rng.random((rows, d)) < 0.5, -1, 1).astype(np.int8)
        obj.evaluate_block(signs)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            obj.evaluate_block(signs)
            ts.append(time.perf_counter() - t0)
        ms = 1e3 * float(np.median(ts))
        print(json.dumps({"shape": tag, "rows": rows, "D": d, "n_wl": nwl, "ms": ms,
                          "domain_evals_per_s": rows * d * nwl / (ms * 1e-3),
                          "h2d_GBps_equiv": rows * d / (ms * 1e-3) / 1e9}))


if __name__ == "__main__":
    main()
