"""Host-side precompute of the per-wavelength phase tables the device consumes.

This is setup, not hot path: it runs once per objective on the host and its
output (e1, b, w, hconst, normalisation per pump wavelength) is uploaded to HBM
once.  The arithmetic mirrors the reference exactly so that the uploaded
tables are bit-identical to the ones the reference's numba kernels read
(checked against tests/golden/tables.npz):

* dispersion: Jundt congruent-LiNbO3 Sellmeier with temperature
  (reference physics.py:97-110, 147-181) and the SHG/SFG mismatches
  dk1 = k(L/2) - 2k(L), dk2 = k(L/3) - k(L/2) - k(L) (physics.py:184-197);
* per-domain moment integrals m0, mn, phi with their small-argument series
  (physics.py:224-270);
* tables: e1_j = exp(-i dk1 j t), b_j = exp(-i dk2 j t), w1 = t m0(i dk1 t),
  w12 = (t m0(i dk1 t)) (t m0(i dk2 t)), hconst = t^2 phi(i dk1 t, i dk2 t)
  sum_j e1_j b_j, normalisation L (SHG) or L^2/2 (THG)
  (physics.py:285-293, 325-339).

Lengths are micrometres, wavelengths cross the API in nm.
"""

import cmath
import math
from dataclasses import dataclass, field
from typing import Mapping, NamedTuple

import numpy as np

TWO_PI = 2.0 * np.pi
SERIES_CUTOFF = 0.25  # |x| below which m0 uses its Taylor series
PHI_CUTOFF = 1e-6  # |x1| below which phi uses its expansion in x1
SERIES_TOL = 1e-20

# Jundt, Opt. Lett. 22, 1553 (1997): extraordinary index of congruent LiNbO3.
SELLMEIER_SETS: dict[str, dict[str, float]] = {
    "linbo3_e": {
        "a1": 5.35583, "a2": 0.100473, "a3": 0.20692, "a4": 100.0, "a5": 11.34927,
        "a6": 1.5334e-2, "b1": 4.629e-7, "b2": 3.862e-8, "b3": -0.89e-8, "b4": 2.657e-5,
    },
}
COEFFICIENT_NAMES = ("a1", "a2", "a3", "a4", "a5", "a6", "b1", "b2", "b3", "b4")


class PhaseMismatchPair(NamedTuple):
    """SHG (dk1) and SFG (dk2) phase mismatches in rad/um."""

    dk1: float
    dk2: float


@dataclass(frozen=True)
class DispersionModel:
    """Sellmeier index model n(lambda, T); raises outside its validity range."""

    coefficients: Mapping[str, float]
    temperature_c: float = 25.0
    wavelength_range_um: tuple[float, float] = (0.4, 5.0)

    def __post_init__(self):
        unknown = sorted(set(self.coefficients) - set(COEFFICIENT_NAMES))
        if unknown:
            raise ValueError(f"unknown Sellmeier coefficient names: {unknown}")
        lo, hi = self.wavelength_range_um
        if not 0 < lo < hi:
            raise ValueError(f"invalid wavelength range [{lo}, {hi}] um")

    def coefficient(self, name: str) -> float:
        return float(self.coefficients.get(name, 0.0))

    def mismatches_at(self, pump_nm: float) -> PhaseMismatchPair:
        return phase_mismatches(self, pump_nm)


def default_dispersion(temperature_c: float = 25.0) -> DispersionModel:
    return DispersionModel(SELLMEIER_SETS["linbo3_e"], temperature_c)


def refractive_index(model: DispersionModel, wavelength_um: float) -> float:
    """Extraordinary index; same operation order as the reference Sellmeier form."""
    lo, hi = model.wavelength_range_um
    if wavelength_um < lo:
        raise ValueError(f"wavelength {wavelength_um} um is below the model's valid minimum {lo} um")
    if wavelength_um > hi:
        raise ValueError(f"wavelength {wavelength_um} um is above the model's valid maximum {hi} um")
    k = model.coefficient
    temp = model.temperature_c
    ft = (temp - 24.5) * (temp + 570.82)
    w2 = wavelength_um * wavelength_um
    n2 = k("a1") + k("b1") * ft - k("a6") * w2
    pole1 = k("a3") + k("b3") * ft
    strength1 = k("a2") + k("b2") * ft
    if strength1 != 0.0:
        n2 += strength1 / (w2 - pole1 ** 2)
    strength2 = k("a4") + k("b4") * ft
    if strength2 != 0.0:
        n2 += strength2 / (w2 - k("a5") ** 2)
    if not n2 > 1.0:
        raise ValueError(f"Sellmeier model yields n^2 = {n2} <= 1 at {wavelength_um} um; "
                         "refractive index must exceed 1 inside the valid range")
    return float(np.sqrt(n2))


def _wavenumber(model: DispersionModel, lam_um: float) -> float:
    return TWO_PI * refractive_index(model, lam_um) / lam_um


def phase_mismatches(model: DispersionModel, pump_wavelength_nm: float) -> PhaseMismatchPair:
    lam = pump_wavelength_nm * 1e-3
    k_p = _wavenumber(model, lam)
    k_sh = TWO_PI * refractive_index(model, lam / 2.0) / (lam / 2.0)
    k_th = TWO_PI * refractive_index(model, lam / 3.0) / (lam / 3.0)
    return PhaseMismatchPair(k_sh - 2.0 * k_p, k_th - k_sh - k_p)


@dataclass(frozen=True)
class MismatchTable:
    """Explicit (dk1, dk2) per pump wavelength, standing in for a dispersion model."""

    entries: Mapping[float, PhaseMismatchPair]

    def mismatches_at(self, pump_nm: float) -> PhaseMismatchPair:
        if pump_nm in self.entries:
            return self.entries[pump_nm]
        known = ", ".join(f"{w:g}" for w in sorted(self.entries))
        raise ValueError(f"no mismatch override for pump {pump_nm:g} nm (have: {known})")


# ---------------------------------------------------------------------------
# moment integrals int_0^1 v^n exp(-x v) dv
# ---------------------------------------------------------------------------

def moment0(x: complex) -> complex:
    if abs(x) < SERIES_CUTOFF:
        acc, term, m = 0.0 + 0.0j, 1.0 + 0.0j, 0
        while abs(term) > SERIES_TOL:
            acc += term / (m + 1)
            m += 1
            term *= -x / m
        return acc
    return (1.0 - cmath.exp(-x)) / x


def moment(n: int, x: complex) -> complex:
    if n == 0:
        return moment0(x)
    if abs(x) < 2.0 * SERIES_CUTOFF:
        acc, term, m = 0.0 + 0.0j, 1.0 + 0.0j, 0
        while abs(term) / (n + m + 1) > SERIES_TOL:
            acc += term / (n + m + 1)
            m += 1
            term *= -x / m
        return acc
    decay = cmath.exp(-x)
    val = moment0(x)
    for p in range(1, n + 1):
        val = (p * val - decay) / x
    return val


def cascade_factor(x1: complex, x2: complex) -> complex:
    """(m0(x2) - m0(x1 + x2)) / x1, expanded in x1 near 0."""
    if abs(x1) < PHI_CUTOFF:
        return moment(1, x2) - x1 * moment(2, x2) / 2.0 + (x1 * x1) * moment(3, x2) / 6.0
    return (moment0(x2) - moment0(x1 + x2)) / x1


# ---------------------------------------------------------------------------
# per-wavelength tables
# ---------------------------------------------------------------------------

@dataclass
class WavelengthTables:
    """Everything the device needs for one pump wavelength."""

    process: str  # "thg" | "shg"
    thickness_um: float
    count: int
    mismatch: PhaseMismatchPair
    e1: np.ndarray  # complex128 [count]
    b: np.ndarray | None  # complex128 [count] (thg)
    w: complex  # w12 (thg) or w1 (shg)
    hconst: complex  # 0 for shg
    normalization: float
    extras: dict = field(default_factory=dict)


def _phases(dk: float, z: np.ndarray) -> np.ndarray:
    return np.exp(-1j * dk * z)


def build_tables(process: str, thickness_um: float, count: int, mismatch) -> WavelengthTables:
    t = float(thickness_um)
    n = int(count)
    dk1, dk2 = float(mismatch[0]), float(mismatch[1])
    z = np.arange(n, dtype=np.float64) * t
    e1 = _phases(dk1, z)
    length = n * t
    if process == "shg":
        return WavelengthTables("shg", t, n, PhaseMismatchPair(dk1, dk2), e1, None,
                                t * moment0(1j * dk1 * t), 0j, length)
    if process != "thg":
        raise ValueError(f"process must be 'shg' or 'thg', got {process!r}")
    b = _phases(dk2, z)
    x1 = 1j * dk1 * t
    x2 = 1j * dk2 * t
    w12 = (t * moment0(x1)) * (t * moment0(x2))
    hconst = t * t * cascade_factor(x1, x2) * complex(np.sum(e1 * b))
    return WavelengthTables("thg", t, n, PhaseMismatchPair(dk1, dk2), e1, b, w12, hconst,
                            0.5 * length * length)


def n_domains(crystal_length_um: float, thickness_um: float) -> int:
    ratio = crystal_length_um / thickness_um
    n = round(ratio)
    if abs(ratio - n) > 1e-9 or n < 1:
        raise ValueError(f"crystal length / domain thickness = {ratio!r} is not an integer domain count")
    return int(n)


def cos_envelope(f_min: float, f_max: float, g: int, total: int) -> float:
    """f_min + (f_max - f_min) cos(pi g / 2G) with Python's libm cos (optimizer.py:290)."""
    progress = g / total if total > 0 else 0.0
    return f_min + (f_max - f_min) * math.cos(0.5 * math.pi * progress)


@dataclass(frozen=True)
class DomainPattern:
    """Equal-thickness +/-1 domain sequence (reference physics.py:43-83)."""

    thickness_um: float
    signs: np.ndarray

    def __post_init__(self):
        if not self.thickness_um > 0:
            raise ValueError(f"domain thickness must be > 0, got {self.thickness_um}")
        raw = np.asarray(self.signs)
        if raw.ndim != 1 or raw.size < 1:
            raise ValueError("signs must be a non-empty 1-d sequence")
        s8 = raw.astype(np.int8)
        if not np.array_equal(s8, raw) or not np.all(np.abs(s8) == 1):
            raise ValueError("every domain sign must be exactly +1 or -1")
        s8.setflags(write=False)
        object.__setattr__(self, "signs", s8)

    @property
    def count(self) -> int:
        return int(self.signs.size)

    @property
    def length_um(self) -> float:
        return self.count * self.thickness_um

    def flipped(self) -> "DomainPattern":
        return DomainPattern(self.thickness_um, -self.signs)
