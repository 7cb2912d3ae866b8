"""Batched |d_eff| spectra on the device (drop-in for physics.sweep_spectrum,
/root/reference/pkg/src/qpmdesign/physics.py:378-395).

The reference builds the phase tables exp(-i dk z) of every wavelength on the
host and scores one pattern per wavelength.  Here the per-wavelength scalars
(dk from the dispersion provider, w = t m0(i dk t) products, the cascade
factor) come from the same host code as the reference (tables.py), and the
O(D) tables are generated inside the kernel (`qpm_sweep_spectrum`), one CTA
per (wavelength, pattern), so many wavelengths and many patterns are scored
in one launch without uploading tables.  Device sincos differs from libm by at
most 1 ulp per phase: |d_eff| agrees with the reference to ~1e-12 relative
(tested against fixtures made by the reference).
"""

import ctypes

import numpy as np

from . import _native
from .tables import DomainPattern, cascade_factor, moment0

PROCESS_IDS = {"shg": _native.QPM_PROCESS_SHG, "thg": _native.QPM_PROCESS_THG}


def _wavelength_scalars(provider, wavelengths_nm, thickness_um: float, process: str):
    t = float(thickness_um)
    M = len(wavelengths_nm)
    dk = np.empty((M, 2), dtype=np.float64)
    w = np.empty((M, 2), dtype=np.float64)
    hphi = np.zeros((M, 2), dtype=np.float64)
    for m, wl in enumerate(wavelengths_nm):
        pair = provider.mismatches_at(wl)
        dk1, dk2 = float(pair[0]), float(pair[1])
        dk[m] = (dk1, dk2)
        x1 = 1j * dk1 * t
        if process == "shg":
            wm = t * moment0(x1)
        else:
            x2 = 1j * dk2 * t
            wm = (t * moment0(x1)) * (t * moment0(x2))
            hp = t * t * cascade_factor(x1, x2)
            hphi[m] = (hp.real, hp.imag)
        w[m] = (wm.real, wm.imag)
    return dk, w, hphi


def sweep_spectra(signs2d, thickness_um: float, provider, wavelengths_nm, process: str) -> np.ndarray:
    """|d_eff| of P patterns (int8 [P, D] of +/-1) at M wavelengths -> f64 [P, M]."""
    if process not in PROCESS_IDS:
        raise ValueError(f"process must be 'shg' or 'thg', got {process!r}")
    signs = np.ascontiguousarray(np.atleast_2d(np.asarray(signs2d)).astype(np.int8))
    P, D = signs.shape
    wls = [float(w) for w in wavelengths_nm]
    out = np.empty((P, len(wls)), dtype=np.float64)
    if not wls:
        return out
    _native.require_cuda()
    dk, w, hphi = _wavelength_scalars(provider, wls, thickness_um, process)
    _native.check(_native.lib().qpm_sweep_spectrum(PROCESS_IDS[process], float(thickness_um), D,
                                                   signs.ctypes.data, P, dk.ctypes.data, w.ctypes.data,
                                                   hphi.ctypes.data, len(wls), out.ctypes.data),
                  "qpm_sweep_spectrum")
    return out


def sweep_spectrum(pattern: DomainPattern, provider, wavelengths_nm, process: str) -> list[tuple[float, float, float]]:
    """(wavelength_nm, |d_eff|, |d_eff| / (L for shg, L^2/2 for thg)) per wavelength, in input order."""
    if process not in PROCESS_IDS:
        raise ValueError(f"process must be 'shg' or 'thg', got {process!r}")
    wls = [float(w) for w in wavelengths_nm]
    mags = sweep_spectra(pattern.signs[None], pattern.thickness_um, provider, wls, process)[0]
    length = pattern.count * float(pattern.thickness_um)
    norm = length if process == "shg" else 0.5 * length * length
    return [(wl, float(mag), float(mag) / norm) for wl, mag in zip(wls, mags)]
