"""ctypes front end of the CPU oracle (oracle/qpm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
reported CPU baseline, never on the product path.

Parity: pinned against vectors produced by the reference package itself
(tests/golden/make_golden.py).  Tables (e1, b, w, hconst) are inputs; the
oracle does not recompute physics.
"""

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libqpm_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, no GPU needed)."""
    src = os.path.join(_HERE, "qpm_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class _Problem(ctypes.Structure):
    _fields_ = [
        ("process", ctypes.c_int),
        ("multi", ctypes.c_int),
        ("n_wl", ctypes.c_int),
        ("D", ctypes.c_int64),
        ("e1", ctypes.c_void_p),
        ("b", ctypes.c_void_p),
        ("w", ctypes.c_void_p),
        ("hconst", ctypes.c_void_p),
        ("scale", ctypes.c_double),
        ("g0", ctypes.c_double),
        ("beta", ctypes.c_double),
    ]


class _Params(ctypes.Structure):
    _fields_ = [
        ("algorithm", ctypes.c_int),
        ("NP", ctypes.c_int64),
        ("D", ctypes.c_int64),
        ("G", ctypes.c_int64),
        ("seed", ctypes.c_int64),
        ("f_max", ctypes.c_double),
        ("f_min", ctypes.c_double),
        ("cr", ctypes.c_double),
        ("x_min", ctypes.c_double),
        ("x_max", ctypes.c_double),
        ("gwo_a", ctypes.c_double),
        ("gwo_a_final", ctypes.c_double),
        ("leader_count", ctypes.c_int),
        ("discreteness_factor", ctypes.c_double),
        ("divide_by_leader_count", ctypes.c_int),
        ("p_dist0", ctypes.c_double),
        ("p_sl0", ctypes.c_double),
        ("p_flip0", ctypes.c_double),
        ("phase_split", ctypes.c_double),
        ("decay_strength", ctypes.c_double),
        ("theta_low_frac", ctypes.c_double),
        ("theta_high_frac", ctypes.c_double),
        ("range_trigger_frac", ctypes.c_double),
        ("explore_boost", ctypes.c_double),
        ("exploit_factor", ctypes.c_double),
        ("conv_threshold", ctypes.c_double),
        ("conv_window", ctypes.c_int),
        ("adaptive_branches", ctypes.c_int),
        ("gwo_lo", ctypes.c_double),
        ("gwo_hi", ctypes.c_double),
        ("threads", ctypes.c_int),
        ("stop_after", ctypes.c_int64),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.qpo_fold_key.restype = ctypes.c_uint64
        L.qpo_fold_key.argtypes = [ctypes.c_int64, ctypes.c_int, P]
        L.qpo_uniform_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, P]
        L.qpo_pairwise_sum.restype = ctypes.c_double
        L.qpo_pairwise_sum.argtypes = [P, ctypes.c_int64, ctypes.c_int64]
        L.qpo_mean_std.argtypes = [P, ctypes.c_int64, P, P, P]
        L.qpo_thg_sum.argtypes = [P, ctypes.c_int64, P, P, P]
        L.qpo_shg_sum.argtypes = [P, ctypes.c_int64, P, P]
        L.qpo_evaluate_block.argtypes = [ctypes.POINTER(_Problem), P, ctypes.c_int64, P, ctypes.c_int]
        L.qpo_sum_block.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int, P, ctypes.c_int64, P]
        L.qpo_reduce_best.argtypes = [P, ctypes.c_int64, ctypes.c_int, P]
        L.qpo_de_pick.restype = ctypes.c_int64
        L.qpo_de_pick.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, P]
        L.qpo_de_trial.restype = ctypes.c_int64
        L.qpo_de_trial.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, P,
                                   ctypes.c_double, ctypes.c_double, P, P, P]
        L.qpo_gwo_discrete.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, P,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int, P]
        L.qpo_gwo_continuous.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, P, P,
                                         ctypes.c_double, ctypes.c_int, P]
        L.qpo_init_population.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_int64, P]
        L.qpo_run.restype = ctypes.c_int64
        L.qpo_run.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(_Params), P, P, P, P]
        L.qpo_run_timed.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(_Params), P, P, P, P, P]
        L.qpo_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _wrap_seed(seed: int) -> int:
    """Python-int seed masked to 64 bits, as a signed int64 for ctypes."""
    s = seed & ((1 << 64) - 1)
    return s - (1 << 64) if s >= (1 << 63) else s


# ---------------------------------------------------------------------------
# RNG
# ---------------------------------------------------------------------------

def fold_key(seed: int, *path: int) -> int:
    arr = np.array([_wrap_seed(p) for p in path], dtype=np.int64)
    return int(lib().qpo_fold_key(_wrap_seed(seed), len(path), _ptr(arr)))


def uniform_fill(key: int, start: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().qpo_uniform_fill(key & ((1 << 64) - 1), start, n, _ptr(out))
    return out


def random_population_matrix(rows: int, n: int, seed: int = 0) -> np.ndarray:
    """bench.random_population_matrix (bench.py:216-218)."""
    u = uniform_fill(fold_key(seed, 0), 0, rows * n)
    return np.where(u < 0.5, -1, 1).astype(np.int8).reshape(rows, n)


def pairwise_sum(a: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().qpo_pairwise_sum(_ptr(a), a.size, 1))


def mean_std(a: np.ndarray):
    a = np.ascontiguousarray(a, dtype=np.float64)
    m = np.zeros(1)
    s = np.zeros(1)
    scratch = np.empty(a.size)
    lib().qpo_mean_std(_ptr(a), a.size, _ptr(m), _ptr(s), _ptr(scratch))
    return float(m[0]), float(s[0])


# ---------------------------------------------------------------------------
# problems (one PatternObjective)
# ---------------------------------------------------------------------------

@dataclass
class Problem:
    """Tables of one objective.  e1, b: complex128 [n_wl, D]; w, hconst: [n_wl]."""

    process: str  # "thg" | "shg"
    e1: np.ndarray
    b: np.ndarray | None
    w: np.ndarray
    hconst: np.ndarray | None
    scale: float = 1.0
    multi: bool = False
    g0: float = 2.0
    beta: float = 1.0
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n_wl(self) -> int:
        return int(np.atleast_2d(self.e1).shape[0])

    @property
    def D(self) -> int:
        return int(np.atleast_2d(self.e1).shape[1])

    def c_struct(self) -> _Problem:
        e1 = np.ascontiguousarray(np.atleast_2d(self.e1), dtype=np.complex128)
        b = (np.ascontiguousarray(np.atleast_2d(self.b), dtype=np.complex128)
             if self.b is not None else np.zeros_like(e1))
        w = np.ascontiguousarray(np.atleast_1d(self.w), dtype=np.complex128)
        h = (np.ascontiguousarray(np.atleast_1d(self.hconst), dtype=np.complex128)
             if self.hconst is not None else np.zeros_like(w))
        self._keep = [e1, b, w, h]
        return _Problem(1 if self.process == "thg" else 0, 1 if self.multi else 0, e1.shape[0], e1.shape[1],
                        e1.ctypes.data, b.ctypes.data, w.ctypes.data, h.ctypes.data,
                        float(self.scale), float(self.g0), float(self.beta))


def evaluate_block(problem: Problem, signs2d: np.ndarray, threads: int = 0) -> np.ndarray:
    signs2d = np.ascontiguousarray(signs2d, dtype=np.int8)
    rows = signs2d.shape[0]
    out = np.empty(rows, dtype=np.float64)
    cs = problem.c_struct()
    lib().qpo_evaluate_block(ctypes.byref(cs), _ptr(signs2d), rows, _ptr(out), threads)
    return out


def sum_block(problem: Problem, signs2d: np.ndarray, wl: int = 0) -> np.ndarray:
    """Complex kernel sums per row (thg_block / shg_block)."""
    signs2d = np.ascontiguousarray(signs2d, dtype=np.int8)
    out = np.empty(signs2d.shape[0], dtype=np.complex128)
    cs = problem.c_struct()
    lib().qpo_sum_block(ctypes.byref(cs), wl, _ptr(signs2d), signs2d.shape[0], _ptr(out))
    return out


def reduce_best(values, k: int) -> list[int]:
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty(k, dtype=np.int64)
    lib().qpo_reduce_best(_ptr(v), v.size, k, _ptr(out))
    return [int(i) for i in out]


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------

def de_trial(key: int, genome: np.ndarray, i: int, f: float, cr: float):
    """Returns (trial f64[D], picks (r1, r2, r3), m, j_rand)."""
    genome = np.ascontiguousarray(genome, dtype=np.float64)
    NP, D = genome.shape
    rows = np.array([genome[r].ctypes.data for r in range(NP)], dtype=np.uint64)
    trial = np.empty(D)
    picks = np.empty(3, dtype=np.int64)
    jr = np.empty(1, dtype=np.int64)
    m = lib().qpo_de_trial(key, NP, D, i, _ptr(rows), f, cr, _ptr(trial), _ptr(picks), _ptr(jr))
    return trial, tuple(int(x) for x in picks), int(m), int(jr[0])


def gwo_discrete(key: int, base: int, leaders: np.ndarray, p_dist: float, p_sl: float, p_flip: float,
                 discreteness: float, early: bool) -> np.ndarray:
    leaders = np.ascontiguousarray(leaders, dtype=np.int8)
    k, D = leaders.shape
    ptrs = np.array([leaders[t].ctypes.data for t in range(k)], dtype=np.uint64)
    out = np.empty(D)
    lib().qpo_gwo_discrete(key, base, D, k, _ptr(ptrs), p_dist, p_sl, p_flip, discreteness, int(early),
                           _ptr(out))
    return out


def gwo_continuous(key: int, x: np.ndarray, leaders: np.ndarray, a: float, divide: bool) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    leaders = np.ascontiguousarray(leaders, dtype=np.float64)
    L, D = leaders.shape
    ptrs = np.array([leaders[t].ctypes.data for t in range(L)], dtype=np.uint64)
    out = np.empty(D)
    lib().qpo_gwo_continuous(key, D, L, _ptr(x), _ptr(ptrs), a, int(divide), _ptr(out))
    return out


def init_population(NP: int, D: int, lo: float, hi: float, seed: int) -> np.ndarray:
    out = np.empty((NP, D))
    lib().qpo_init_population(NP, D, lo, hi, _wrap_seed(seed), _ptr(out))
    return out


# ---------------------------------------------------------------------------
# run drivers
# ---------------------------------------------------------------------------

ALGORITHMS = {"hybrid": 0, "de": 1, "gwo": 2}


@dataclass
class RunSettings:
    """Flat mirror of DEParams / GWOParams / Schedules defaults (optimizer.py:84-173)."""

    f_max: float = 0.1
    f_min: float = 0.01
    cr: float = 0.9
    x_min: float = -1.0
    x_max: float = 1.0
    gwo_a: float = 2.0
    gwo_a_final: float = 0.0
    leader_count: int = 4
    discreteness_factor: float = 1.0
    divide_by_leader_count: bool = False
    p_dist0: float = 0.1
    p_sl0: float = 0.05
    p_flip0: float = 0.02
    phase_split: float = 0.5
    decay_strength: float = 0.2
    theta_low_frac: float = 0.05
    theta_high_frac: float = 0.5
    range_trigger_frac: float = 1.0
    explore_boost: float = 1.2
    exploit_factor: float = 0.8
    conv_threshold: float = 0.1
    conv_window: int = 10
    adaptive_branches: bool = True
    gwo_lo: float = -1.0
    gwo_hi: float = 1.0


def run(problem: Problem, algorithm: str, NP: int, G: int, seed: int, settings: RunSettings | None = None,
        threads: int = 0, stop_after: int = -1, gen_end_s: np.ndarray | None = None):
    """Returns (trace [rows, 5], best_genome, best_proj, best_fit).  gen_end_s
    (float64 [G+1], optional) receives the monotonic time at which each
    generation's trace row was complete (benchmark windows inside one run)."""
    s = settings or RunSettings()
    D = problem.D
    p = _Params(ALGORITHMS[algorithm], NP, D, G, _wrap_seed(seed), s.f_max, s.f_min, s.cr, s.x_min, s.x_max,
                s.gwo_a, s.gwo_a_final, s.leader_count, s.discreteness_factor, int(s.divide_by_leader_count),
                s.p_dist0, s.p_sl0, s.p_flip0, s.phase_split, s.decay_strength, s.theta_low_frac,
                s.theta_high_frac, s.range_trigger_frac, s.explore_boost, s.exploit_factor,
                s.conv_threshold, s.conv_window, int(s.adaptive_branches), s.gwo_lo, s.gwo_hi, threads,
                stop_after)
    trace = np.zeros((G + 1, 5))
    bg = np.empty(D)
    bp = np.empty(D, dtype=np.int8)
    bf = np.empty(1)
    cs = problem.c_struct()
    if gen_end_s is not None:
        assert gen_end_s.dtype == np.float64 and gen_end_s.size >= G + 1
        n = lib().qpo_run_timed(ctypes.byref(cs), ctypes.byref(p), _ptr(trace), _ptr(bg), _ptr(bp), _ptr(bf),
                                _ptr(gen_end_s))
    else:
        n = lib().qpo_run(ctypes.byref(cs), ctypes.byref(p), _ptr(trace), _ptr(bg), _ptr(bp), _ptr(bf))
    return trace[:n], bg, bp, float(bf[0])


def max_threads() -> int:
    return int(lib().qpo_max_threads())
