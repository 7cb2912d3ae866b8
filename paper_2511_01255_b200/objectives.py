"""Fitness objectives evaluated on the B200 (drop-in for objectives.py).

`make_objective(spec, provider, thickness_um, count)` returns a
`GpuPatternObjective` with the reference PatternObjective's protocol
(objectives.py:72-123): `__call__(signs)`, `evaluate_block(signs2d)`,
`gains`, `normalized_gains`, `dimension`.  It can be handed to the
reference's own optimizer (plug point 1 of SURVEY.md §8(b)) or to this
package's device-resident `run_*` drivers, which use its device tables
directly.

Fitness is maximised.  Multi-wavelength variants score
f = sum_i |G0 - G_i| + beta (G_max - G_min) and return -f.
"""

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .tables import build_tables

VARIANTS = ("single_shg", "single_thg", "multi_shg", "multi_thg")
MODES = {"fast": _native.QPM_MODE_FAST, "exact": _native.QPM_MODE_EXACT}


@dataclass(frozen=True)
class ObjectiveSpec:
    """Process, pump wavelengths and scoring (objectives.py:23-63)."""

    variant: str
    pump_wavelengths_nm: tuple[float, ...]
    g0: float = 2.0
    beta: float = 1.0
    normalization: str = "normalized"

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"variant must be one of {VARIANTS}, got {self.variant!r}")
        pumps = tuple(float(w) for w in self.pump_wavelengths_nm)
        object.__setattr__(self, "pump_wavelengths_nm", pumps)
        if not pumps:
            raise ValueError("pump_wavelengths_nm must be non-empty")
        if self.is_multi:
            if len(pumps) < 2:
                raise ValueError("multi variants need at least 2 pump wavelengths")
            if not self.g0 > 0:
                raise ValueError("g0 must be > 0 for multi variants")
        elif len(pumps) != 1:
            raise ValueError("single variants take exactly 1 pump wavelength")
        if self.beta < 0:
            raise ValueError("beta must be >= 0")
        if self.normalization not in ("normalized", "raw"):
            raise ValueError("normalization must be 'normalized' or 'raw'")

    @property
    def is_multi(self) -> bool:
        return self.variant.startswith("multi")

    @property
    def process(self) -> str:
        return "shg" if self.variant.endswith("shg") else "thg"


def multi_objective(gains: Sequence[float], g0: float, beta: float) -> float:
    g = np.asarray(gains, dtype=np.float64)
    return float(np.sum(np.abs(g0 - g)) + beta * (np.max(g) - np.min(g)))


def _interleave(z: np.ndarray) -> np.ndarray:
    z = np.ascontiguousarray(z, dtype=np.complex128)
    return z.view(np.float64)


class GpuPatternObjective:
    """Device-resident fitness of +/-1 domain patterns for one geometry/spec.

    mode="fast" (default) uses the FP64 quad-table scan (<= 1e-9 relative of
    the reference, ~1e-14 in practice); mode="exact" replays numba's
    sequential arithmetic and is bit-identical to the reference.
    """

    def __init__(self, spec: ObjectiveSpec, provider, thickness_um: float, count: int, mode: str = "fast",
                 seg_chunks: int | None = None):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {tuple(MODES)}, got {mode!r}")
        if seg_chunks is not None and int(seg_chunks) < 1:
            raise ValueError(f"seg_chunks must be >= 1, got {seg_chunks}")
        self._seg_req = int(seg_chunks or 0)  # 0: the library's default for D and the wavelength count
        self.spec = spec
        self.thickness_um = float(thickness_um)
        self.count = int(count)
        self.mode = mode
        pairs = [provider.mismatches_at(wl) for wl in spec.pump_wavelengths_nm]
        self.tables = [build_tables(spec.process, self.thickness_um, self.count, pair) for pair in pairs]
        self._scale = self.tables[0].normalization if spec.normalization == "normalized" else 1.0
        self._handle = None
        self._create()

    # -- device problem -------------------------------------------------
    def _create(self):
        _native.require_cuda()
        L = _native.lib()
        thg = self.spec.process == "thg"
        e1 = _interleave(np.stack([t.e1 for t in self.tables]))
        b = _interleave(np.stack([t.b for t in self.tables])) if thg else None
        w = _interleave(np.array([t.w for t in self.tables]))
        h = _interleave(np.array([t.hconst for t in self.tables])) if thg else None
        self._keep = (e1, b, w, h)
        import ctypes

        handle = ctypes.c_void_p()
        _native.check(L.qpm_problem_create(
            ctypes.byref(handle), _native.QPM_PROCESS_THG if thg else _native.QPM_PROCESS_SHG,
            1 if self.spec.is_multi else 0, len(self.tables), self.count, e1.ctypes.data,
            b.ctypes.data if b is not None else None, w.ctypes.data, h.ctypes.data if h is not None else None,
            float(self._scale), float(self.spec.g0), float(self.spec.beta), self._seg_req), "qpm_problem_create")
        self._handle = handle
        self.row_words = int(L.qpm_problem_row_words(handle))
        sc, S, nsb = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _native.check(L.qpm_problem_layout(handle, ctypes.byref(sc), ctypes.byref(S), ctypes.byref(nsb)),
                      "qpm_problem_layout")
        # fast-scan layout: segment length (128-domain chunks), segments, stitch super-blocks
        self.seg_chunks, self.segments, self.super_blocks = sc.value, S.value, nsb.value

    @property
    def handle(self):
        return self._handle

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _native.lib().qpm_problem_destroy(h)
            except Exception:
                pass
            self._handle = None

    # -- reference protocol ---------------------------------------------
    @property
    def dimension(self) -> int:
        return self.count

    @property
    def normalization(self) -> float:
        return self._scale

    def _mode_id(self, mode):
        return MODES[mode or self.mode]

    def evaluate_block(self, signs2d: np.ndarray, mode: str | None = None) -> np.ndarray:
        """f64[rows] for an int8 [rows, D] matrix (host in, host out)."""
        signs2d = np.ascontiguousarray(signs2d, dtype=np.int8)
        if signs2d.ndim != 2 or signs2d.shape[1] != self.count:
            raise ValueError(f"signs2d must have shape (rows, {self.count}), got {signs2d.shape}")
        rows = signs2d.shape[0]
        out = np.empty(rows, dtype=np.float64)
        if rows == 0:
            return out
        _native.check(_native.lib().qpm_evaluate_block_host(self._handle, signs2d.ctypes.data, rows,
                                                            out.ctypes.data, self._mode_id(mode)),
                      "qpm_evaluate_block_host")
        return out

    def __call__(self, signs: np.ndarray) -> float:
        return float(self.evaluate_block(np.asarray(signs)[np.newaxis, :])[0])

    def kernel_sums(self, signs2d: np.ndarray, wl: int = 0) -> np.ndarray:
        """Complex kernel sums (the reference's thg_block / shg_block), exact order."""
        signs2d = np.ascontiguousarray(signs2d, dtype=np.int8)
        out = np.empty(signs2d.shape[0], dtype=np.complex128)
        _native.check(_native.lib().qpm_sum_block_host(self._handle, wl, signs2d.ctypes.data, signs2d.shape[0],
                                                       out.ctypes.data), "qpm_sum_block_host")
        return out

    def _abs_deff(self, signs: np.ndarray) -> list[float]:
        vals = []
        row = np.asarray(signs, dtype=np.int8)[np.newaxis, :]
        for wl, t in enumerate(self.tables):
            acc = complex(self.kernel_sums(row, wl)[0])
            z = t.w * acc + t.hconst if t.process == "thg" else acc * t.w
            vals.append(abs(z))
        return vals

    def gains(self, signs: np.ndarray) -> np.ndarray:
        return np.array([v / self._scale for v in self._abs_deff(signs)])

    def normalized_gains(self, signs: np.ndarray) -> np.ndarray:
        return np.array([v / t.normalization for v, t in zip(self._abs_deff(signs), self.tables)])

    # -- device-level entry point ---------------------------------------
    def evaluate_bits(self, bits, out, row_index=None, stream=None, mode: str | None = None):
        """Fitness of bit-packed CUDA rows (uint32/int32 [*, row_words]) into `out` (f64 CUDA)."""
        rows = int(out.numel()) if row_index is None else int(row_index.numel())
        _native.check(_native.lib().qpm_fitness_bits(
            self._handle, bits.data_ptr(), self.row_words,
            row_index.data_ptr() if row_index is not None else None, rows, out.data_ptr(),
            self._mode_id(mode), _native.stream_handle(stream)), "qpm_fitness_bits")
        return out


PatternObjective = GpuPatternObjective


def make_objective(spec: ObjectiveSpec, provider, thickness_um: float, count: int,
                   mode: str = "fast", seg_chunks: int | None = None) -> GpuPatternObjective:
    """objectives.make_objective (objectives.py:126-130) on the device; seg_chunks
    optionally fixes the fast scan's segment length (multi-GPU runs pick one
    whose segments split evenly over their ranks)."""
    return GpuPatternObjective(spec, provider, thickness_um, count, mode=mode, seg_chunks=seg_chunks)


def fitness_single(pattern, spec: ObjectiveSpec, provider, mode: str = "fast") -> float:
    if spec.is_multi:
        raise ValueError(f"fitness_single requires a single_* variant, got {spec.variant!r}")
    return GpuPatternObjective(spec, provider, pattern.thickness_um, pattern.count, mode)(pattern.signs)


def fitness_multi(pattern, spec: ObjectiveSpec, provider, mode: str = "fast") -> float:
    if not spec.is_multi:
        raise ValueError(f"fitness_multi requires a multi_* variant, got {spec.variant!r}")
    return GpuPatternObjective(spec, provider, pattern.thickness_um, pattern.count, mode)(pattern.signs)
