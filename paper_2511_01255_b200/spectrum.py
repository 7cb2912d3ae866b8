"""Batched |d_eff| spectra on the device (drop-in for physics.sweep_spectrum,
/root/reference/pkg/src/qpmdesign/physics.py:378-395).

The reference builds the phase tables exp(-i dk z) of every wavelength on the
host and scores one pattern per wavelength.  Here the per-wavelength scalars
(dk from the dispersion provider, w = t m0(i dk t) products, the cascade
factor) are computed on the device for a Sellmeier model
(`qpm_wavelength_scalars`: dk bit-identical to tables.py, w and the cascade
factor within ~1e-16) or taken from an explicit mismatch table, and the
O(D) tables are generated inside the kernel (`qpm_sweep_spectrum`), one CTA
per (wavelength, pattern), so many wavelengths and many patterns are scored
in one launch without uploading tables.  Device sincos differs from libm by at
most 1 ulp per phase: |d_eff| agrees with the reference to ~1e-12 relative
(tested against fixtures made by the reference).
"""

import ctypes

import numpy as np

from . import _native
from .tables import DispersionModel, DomainPattern, cascade_factor, moment0, phase_mismatches

PROCESS_IDS = {"shg": _native.QPM_PROCESS_SHG, "thg": _native.QPM_PROCESS_THG}


def _sellmeier_terms(model: DispersionModel) -> np.ndarray:
    """The wavelength-free terms of tables.refractive_index, with Python's own
    arithmetic (its pole**2 is libm pow): the device finishes n(lambda) from
    them bit for bit."""
    k = model.coefficient
    temp = model.temperature_c
    ft = (temp - 24.5) * (temp + 570.82)
    return np.array([k("a1") + k("b1") * ft, k("a6"), k("a2") + k("b2") * ft, (k("a3") + k("b3") * ft) ** 2,
                     k("a4") + k("b4") * ft, k("a5") ** 2], dtype=np.float64)


def _device_wavelength_scalars(model: DispersionModel, wavelengths_nm, thickness_um: float, process: str):
    """(dk, w, hphi) [M, 2] of a Sellmeier model computed on the device
    (qpm_wavelength_scalars): dk bit-identical to the host loop, w / hphi to
    ~1e-16.  Out-of-range wavelengths raise the reference's ValueError."""
    wls = np.asarray(wavelengths_nm, dtype=np.float64)
    lo, hi = model.wavelength_range_um
    lam = wls * 1e-3
    bad = (lam < lo) | (lam > hi) | (lam / 2.0 < lo) | (lam / 2.0 > hi) | (lam / 3.0 < lo) | (lam / 3.0 > hi)
    if bad.any():  # the host formula raises the reference's message for the first offending wavelength
        phase_mismatches(model, float(wls[int(np.argmax(bad))]))
    M = len(wls)
    dk = np.empty((M, 2))
    w = np.empty((M, 2))
    hphi = np.empty((M, 2))
    bad_index = ctypes.c_int64(-1)
    terms = _sellmeier_terms(model)
    rc = _native.lib().qpm_wavelength_scalars(PROCESS_IDS[process], float(thickness_um), terms.ctypes.data,
                                              wls.ctypes.data, M, dk.ctypes.data, w.ctypes.data, hphi.ctypes.data,
                                              ctypes.byref(bad_index))
    if rc == _native.QPM_ERR_ARG and bad_index.value >= 0:
        phase_mismatches(model, float(wls[bad_index.value]))  # raises the reference's n^2 <= 1 message
    _native.check(rc, "qpm_wavelength_scalars")
    return dk, w, hphi


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
    if isinstance(provider, DispersionModel):  # Sellmeier and moment integrals on the device
        dk, w, hphi = _device_wavelength_scalars(provider, wls, thickness_um, process)
    else:  # explicit mismatch tables: the provider's own values
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
