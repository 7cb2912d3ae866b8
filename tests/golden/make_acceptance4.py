"""Record the reference's acceptance criterion 4 trials (algorithm ordering,
/root/reference/pkg/tests/test_acceptance.py:103-142) by running the
reference package itself:

    python tests/golden/make_acceptance4.py

Desk-scale table analog: L = 660 um at t = 1 um (660 domains) and t = 0.5 um
(1320 domains), single_thg at 1404 nm, NP 200, 300 generations,
gwo_a 0.1 -> 0.01, 10 trials with seeds 100..109, hybrid / DE / GWO (GWO at
660 only).  Writes tests/golden/acceptance4.npz with every trial's final
fitness, best projection (bit-packed) and the reference's per-(label,
algorithm) means; the GPU test re-runs the same trials in exact mode and must
reproduce them bit-for-bit, then checks the criterion itself.
"""

import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

from qpmdesign import _kernels, bench  # noqa: E402
from qpmdesign.config import parse_config_text  # noqa: E402

assert _kernels.backend() == "numba"

TABLE_CFG = """
crystal_length_um = 660
domain_thickness_um = {thickness}
process = single_thg
pump_wavelengths_nm = 1404
np = 200
generations = 300
gwo_a_initial = 0.1
gwo_a_final = 0.01
workers = 2
"""
TRIALS, BASE_SEED = 10, 100


def main():
    out = {}
    cases = []
    t0 = time.perf_counter()
    for label, thick, algos in (("660", 1, ("hybrid", "de", "gwo")), ("1320", 0.5, ("hybrid", "de"))):
        cfg = parse_config_text(TABLE_CFG.format(thickness=thick))
        for algo in algos:
            stats, records = bench.run_trials(cfg, algo, TRIALS, BASE_SEED)
            key = f"{label}_{algo}"
            cases.append({"key": key, "label": label, "algorithm": algo, "thickness": thick,
                          "n_domains": cfg.n_domains})
            out[f"{key}__final"] = np.array([r.final_fitness for r in records])
            out[f"{key}__seeds"] = np.array([r.seed for r in records])
            out[f"{key}__mean"] = np.array(stats.average)
            print(key, stats.average, f"{time.perf_counter() - t0:.0f}s", flush=True)
    out["cases"] = np.array(json.dumps(cases))
    out["meta"] = np.array("qpmdesign.bench.run_trials (test_acceptance.py:103-142 configs), numba backend")
    path = os.path.join(HERE, "acceptance4.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
