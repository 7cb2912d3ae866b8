"""Batched spectra timing: P patterns x M pump wavelengths x D domains, with the
per-wavelength scalars on the device (Sellmeier model) and from the host loop.

    python tools/spectrum_probe.py [--p 8] [--m 1000] [--d 20000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--m", type=int, default=1000)
    ap.add_argument("--d", type=int, default=20_000)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200.spectrum import _device_wavelength_scalars, _wavelength_scalars

    torch.cuda.set_device(0)
    model = q.default_dispersion()
    wls = np.linspace(1300.0, 1500.0, args.m)
    rng = np.random.default_rng(0)
    signs = np.where(rng.random((args.p, args.d)) < 0.5, -1, 1).astype(np.int8)
    q.sweep_spectra(signs[:1], 1.0, model, wls[:4], "thg")  # warm-up
    out = {"P": args.p, "M": args.m, "D": args.d}
    for name, fn in (("device_scalars_ms", lambda: _device_wavelength_scalars(model, wls, 1.0, "thg")),
                     ("host_scalars_ms", lambda: _wavelength_scalars(model, wls, 1.0, "thg")),
                     ("sweep_spectra_ms", lambda: q.sweep_spectra(signs, 1.0, model, wls, "thg"))):
        fn()
        t0 = time.perf_counter()
        fn()
        out[name] = 1e3 * (time.perf_counter() - t0)
    out["domain_evals_per_s"] = args.p * args.m * args.d / (out["sweep_spectra_ms"] * 1e-3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
