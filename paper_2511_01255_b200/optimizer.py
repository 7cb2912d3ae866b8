"""HWSDA run drivers on the B200 (drop-in for the reference's optimizer.py).

`run(algorithm, objective, *, dimension, pop_size, generations, seed, ...)`
and `run_hybrid` / `run_de` / `run_gwo` keep the reference's keywords,
validation errors and `RunResult(best, trace)` semantics (optimizer.py:400-616)
but execute the whole population loop on the device: the population lives in
HBM, every generation is one CUDA-graph replay of the native engine
(libqpm_b200.so, include/qpm_b200.h), and the host only reads the trace and
the best individual back at the end.

The per-generation scalars that the reference computes with Python floats
(cosine F envelope, damping, schedule rates, the early-phase flag, GWO's a)
are computed here with the same Python expressions and uploaded once, so the
device makes the same decisions.  With `fitness_mode="exact"` the traces are
bit-identical to the reference's; the default "fast" mode differs only by
fitness rounding (~1e-14 relative).
"""

import ctypes
import math
from dataclasses import astuple, dataclass, replace

import numpy as np

from . import _native
from .objectives import GpuPatternObjective

ALGORITHMS = ("hybrid", "de", "gwo")


# ---------------------------------------------------------------------------
# data types (optimizer.py:39-200)
# ---------------------------------------------------------------------------

@dataclass
class Individual:
    genome: np.ndarray
    projection: np.ndarray
    fitness: float | None = None

    @classmethod
    def from_genome(cls, genome: np.ndarray, fitness: float | None = None) -> "Individual":
        genome = np.ascontiguousarray(genome, dtype=np.float64)
        return cls(genome=genome, projection=np.where(genome >= 0.0, 1, -1).astype(np.int8), fitness=fitness)


@dataclass
class Population:
    individuals: list
    generation: int = 0
    rng_seed: int = 0

    def __post_init__(self):
        if len(self.individuals) < 4:
            raise ValueError(f"population size must be >= 4, got {len(self.individuals)}")

    @property
    def size(self) -> int:
        return len(self.individuals)

    @property
    def dimension(self) -> int:
        return int(self.individuals[0].genome.size)

    def fitness_values(self) -> np.ndarray:
        vals = [ind.fitness for ind in self.individuals]
        if any(v is None for v in vals):
            raise ValueError("population has unevaluated individuals")
        return np.asarray(vals, dtype=np.float64)


@dataclass
class DEParams:
    f: float = 0.1
    cr: float = 0.9
    f_min: float = 0.01
    f_max: float = 0.1
    x_min: float = -1.0
    x_max: float = 1.0

    def __post_init__(self):
        if not (0.0 < self.f_min <= self.f_max <= 2.0):
            raise ValueError(f"need 0 < f_min <= f_max <= 2, got [{self.f_min}, {self.f_max}]")
        if not (0.0 <= self.cr <= 1.0):
            raise ValueError(f"cr must be in [0, 1], got {self.cr}")
        if not (self.f_min <= self.f <= self.f_max):
            raise ValueError(f"f={self.f} outside [{self.f_min}, {self.f_max}]")


@dataclass
class GWOParams:
    a: float = 2.0
    a_final: float = 0.0
    leader_count: int = 4
    p_dist: float = 0.1
    p_sl: float = 0.05
    p_flip: float = 0.02
    discreteness_factor: float = 1.0
    divide_by_leader_count: bool = False

    def __post_init__(self):
        if not (0.0 <= self.a <= 2.0):
            raise ValueError(f"a must be in [0, 2], got {self.a}")
        if not (0.0 <= self.a_final <= self.a):
            raise ValueError(f"a_final must be in [0, a], got {self.a_final}")
        if self.leader_count not in (3, 4):
            raise ValueError(f"leader_count must be 3 or 4, got {self.leader_count}")
        for name in ("p_dist", "p_sl", "p_flip", "discreteness_factor"):
            v = getattr(self, name)
            if not (0.0 <= v <= 1.0):
                raise ValueError(f"{name} must be in [0, 1], got {v}")


@dataclass
class Schedules:
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

    def p_dist(self, g: int, total: int) -> float:
        return self.p_dist0 * (1.0 - g / total) if total else 0.0

    def p_sl(self, g: int, total: int) -> float:
        return self.p_sl0 * (1.0 - g / total) if total else 0.0

    def p_flip(self, g: int, total: int) -> float:
        return self.p_flip0 * (1.0 - g / total) if total else 0.0

    def decay_coeff(self, g: int, total: int) -> float:
        prog = g / total if total else 0.0
        return 1.0 - self.decay_strength * prog * prog

    def is_early(self, g: int, total: int) -> bool:
        return (g / total if total else 0.0) < self.phase_split


@dataclass
class AdaptiveState:
    generation: int
    total_generations: int
    pop_std: float
    fit_range: float
    convergence_rate: float
    decay_coeff: float
    baseline_std: float


def make_trace_row(generation, best, mean, f, pop_std):
    return (int(generation), float(best), float(mean), float(f), float(pop_std))


@dataclass
class RunResult:
    best: Individual
    trace: list

    def trace_column(self, name: str) -> np.ndarray:
        cols = {"generation": 0, "best": 1, "mean": 2, "f": 3, "pop_std": 4}
        return np.array([row[cols[name]] for row in self.trace])


def adaptive_f_update(state: AdaptiveState, params: DEParams, schedules: Schedules) -> float:
    """Host reference of the F rule the stats kernel applies (optimizer.py:277-299)."""
    total = state.total_generations
    progress = state.generation / total if total > 0 else 0.0
    f = params.f_min + (params.f_max - params.f_min) * math.cos(0.5 * math.pi * progress)
    if schedules.adaptive_branches:
        low = schedules.theta_low_frac * state.baseline_std
        high = schedules.theta_high_frac * state.baseline_std
        trig = schedules.range_trigger_frac * state.baseline_std
        if state.pop_std < low or state.convergence_rate < schedules.conv_threshold:
            f *= schedules.explore_boost
        if state.pop_std > high or state.fit_range < trig:
            f *= schedules.exploit_factor
    f *= state.decay_coeff
    return min(max(f, params.f_min), params.f_max)


# ---------------------------------------------------------------------------
# schedule table
# ---------------------------------------------------------------------------

_SCHED_CACHE: dict = {}


def _schedule_cached(generations: int, de: DEParams, gwo: GWOParams, sch: Schedules) -> np.ndarray:
    """schedule_table, memoised on the parameter values (read-only array): batched
    trials and repeated runs of one configuration build it once."""
    key = (int(generations), astuple(de), astuple(gwo), astuple(sch))
    tab = _SCHED_CACHE.get(key)
    if tab is None:
        if len(_SCHED_CACHE) >= 64:
            _SCHED_CACHE.clear()
        tab = np.ascontiguousarray(schedule_table(generations, de, gwo, sch))
        tab.flags.writeable = False
        _SCHED_CACHE[key] = tab
    return tab


def schedule_table(generations: int, de: DEParams, gwo: GWOParams, sch: Schedules) -> np.ndarray:
    """[G+1, 8] per-generation scalars with the reference's float arithmetic.

    Elementwise IEEE operations are done by numpy in the order the reference's
    Python expressions use (bit-identical); the cosine envelope keeps Python's
    math.cos (optimizer.py:290), which numpy's cos may differ from by an ulp."""
    G = int(generations)
    tab = np.zeros((G + 1, _native.SCHED_COLS), dtype=np.float64)
    if G > 0:
        prog = np.arange(G + 1, dtype=np.float64) / float(G)  # g / G, correctly rounded like Python's
    else:
        prog = np.zeros(1)
    cos = np.array([math.cos(0.5 * math.pi * float(p)) for p in prog])
    tab[:, _native.SCHED_F_ENV] = de.f_min + (de.f_max - de.f_min) * cos
    tab[:, _native.SCHED_DECAY] = 1.0 - sch.decay_strength * prog * prog
    if G > 0:
        rest = 1.0 - prog
        tab[:, _native.SCHED_P_DIST] = sch.p_dist0 * rest
        tab[:, _native.SCHED_P_SL] = sch.p_sl0 * rest
        tab[:, _native.SCHED_P_FLIP] = sch.p_flip0 * rest
    tab[:, _native.SCHED_EARLY] = np.where(prog < sch.phase_split, 1.0, 0.0)
    tab[:, _native.SCHED_A_NOW] = gwo.a_final + (gwo.a - gwo.a_final) * (1.0 - prog)
    return tab


def _schedule_table_reference(generations: int, de: DEParams, gwo: GWOParams, sch: Schedules) -> np.ndarray:
    """The same table by the reference's per-generation Python expressions (tests compare the two)."""
    G = int(generations)
    tab = np.zeros((G + 1, _native.SCHED_COLS), dtype=np.float64)
    for g in range(G + 1):
        progress = g / G if G > 0 else 0.0
        tab[g, _native.SCHED_F_ENV] = de.f_min + (de.f_max - de.f_min) * math.cos(0.5 * math.pi * progress)
        tab[g, _native.SCHED_DECAY] = sch.decay_coeff(g, G)
        tab[g, _native.SCHED_P_DIST] = sch.p_dist(g, G)
        tab[g, _native.SCHED_P_SL] = sch.p_sl(g, G)
        tab[g, _native.SCHED_P_FLIP] = sch.p_flip(g, G)
        tab[g, _native.SCHED_EARLY] = 1.0 if sch.is_early(g, G) else 0.0
        gp = g / G if G else 0.0
        tab[g, _native.SCHED_A_NOW] = gwo.a_final + (gwo.a - gwo.a_final) * (1.0 - gp)
    return tab


# ---------------------------------------------------------------------------
# engine wrapper
# ---------------------------------------------------------------------------

_STREAMS: dict = {}  # device index -> idle high-priority streams (reused by later engines)


def _stream_acquire(dev):
    import torch

    free = _STREAMS.setdefault(dev.index, [])
    if free:
        return free.pop()
    return torch.cuda.Stream(dev, priority=min(torch.cuda.Stream.priority_range()))


class Engine:
    """One device-resident run (thin owner of a qpm_engine handle)."""

    def __init__(self, objective: GpuPatternObjective, algorithm: str, *, pop_size: int, generations: int,
                 seed: int, de: DEParams, gwo: GWOParams, sch: Schedules, fitness_mode: str | None = None,
                 bounds: tuple[float, float] = (-1.0, 1.0), stream=None, shard: tuple[int, int] = (0, 1)):
        import torch

        if not isinstance(objective, GpuPatternObjective):
            raise TypeError("the device engine needs a GpuPatternObjective (make_objective of this package); "
                            f"got {type(objective).__name__}")
        dev = _native.require_cuda()
        self.objective = objective
        self.algorithm = algorithm
        self.NP = int(pop_size)
        self.G = int(generations)
        self.D = objective.dimension
        # a dedicated high-priority stream (CUDA graphs cannot be captured on the
        # legacy default stream; the engine's planner runs on a low-priority one)
        self._pooled = stream is None
        if stream is None:
            stream = _stream_acquire(dev)
        self.stream = stream
        mode = fitness_mode or objective.mode
        from .objectives import MODES
        from .rng import signed64

        p = _native.RunParams()
        p.algorithm = _native.QPM_ALGO[algorithm]
        p.fitness_mode = MODES[mode]
        p.NP, p.G, p.seed = self.NP, self.G, signed64(seed)
        p.f_max, p.f_min, p.cr, p.x_min, p.x_max = de.f_max, de.f_min, de.cr, de.x_min, de.x_max
        p.leader_count = gwo.leader_count
        p.discreteness_factor = gwo.discreteness_factor
        p.divide_by_leader_count = int(gwo.divide_by_leader_count)
        p.theta_low_frac, p.theta_high_frac = sch.theta_low_frac, sch.theta_high_frac
        p.range_trigger_frac, p.explore_boost = sch.range_trigger_frac, sch.explore_boost
        p.exploit_factor, p.conv_threshold = sch.exploit_factor, sch.conv_threshold
        p.conv_window = max(1, int(sch.conv_window))
        p.adaptive_branches = int(bool(sch.adaptive_branches))
        p.gwo_lo, p.gwo_hi, p.gwo_a0 = float(bounds[0]), float(bounds[1]), gwo.a
        p.shard_rank, p.shard_world = int(shard[0]), int(shard[1])
        self.params = p
        self.sched = _schedule_cached(self.G, de, gwo, sch)
        h = ctypes.c_void_p()
        _native.check(_native.lib().qpm_engine_create(ctypes.byref(h), objective.handle, ctypes.byref(p),
                                                      self.sched.ctypes.data, self.stream.cuda_stream),
                      "qpm_engine_create")
        self.handle = h
        g0, dl = ctypes.c_int64(), ctypes.c_int64()
        _native.check(_native.lib().qpm_engine_columns(h, ctypes.byref(g0), ctypes.byref(dl)), "qpm_engine_columns")
        # this engine's genes [g0, g0 + Dl): all of them on one GPU, a column shard on several
        self.g0, self.Dl = int(g0.value), int(dl.value)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _native.lib().qpm_engine_destroy(h)  # synchronises the engine's stream
            except Exception:
                pass
            self.handle = None
            if getattr(self, "_pooled", False):
                _STREAMS.setdefault(self.stream.device.index, []).append(self.stream)

    def init(self):
        _native.check(_native.lib().qpm_engine_init(self.handle), "qpm_engine_init")

    def step(self, n: int, use_graph: bool = True):
        _native.check(_native.lib().qpm_engine_step(self.handle, int(n), int(use_graph)), "qpm_engine_step")

    def checkpoint(self) -> bytes:
        """A host snapshot of the run (qpm_engine_checkpoint); restore() it into a new
        Engine created with the same arguments to resume bit-identically."""
        n = int(_native.lib().qpm_engine_checkpoint_bytes(self.handle))
        buf = np.empty(n, dtype=np.uint8)
        _native.check(_native.lib().qpm_engine_checkpoint(self.handle, buf.ctypes.data, n), "qpm_engine_checkpoint")
        return buf.tobytes()

    def restore(self, data: bytes):
        """Resume from checkpoint() bytes (instead of init())."""
        buf = np.frombuffer(data, dtype=np.uint8)
        _native.check(_native.lib().qpm_engine_restore(self.handle, buf.ctypes.data, buf.size), "qpm_engine_restore")

    def prepare(self, n: int):
        """Capture and upload the CUDA graphs a step(n) replays (keeps capture out of timed regions)."""
        _native.check(_native.lib().qpm_engine_prepare(self.handle, int(n)), "qpm_engine_prepare")

    def finalize(self):
        _native.check(_native.lib().qpm_engine_finalize(self.handle), "qpm_engine_finalize")

    def profile(self, n: int) -> list[tuple[str, float]]:
        """Run n generations eagerly with CUDA events between stages; mean ms per stage."""
        ms = np.zeros(16, dtype=np.float64)
        ns = ctypes.c_int()
        names = ctypes.create_string_buffer(16 * 32)
        _native.check(_native.lib().qpm_engine_profile(self.handle, int(n), ms.ctypes.data, ctypes.byref(ns),
                                                       names, 32), "qpm_engine_profile")
        out = []
        for k in range(ns.value):
            out.append((names.raw[k * 32:(k + 1) * 32].split(b"\0", 1)[0].decode(), float(ms[k])))
        return out

    @property
    def launches_per_generation(self) -> int:
        return int(_native.lib().qpm_engine_launches_per_generation(self.handle))

    @property
    def device_bytes(self) -> int:
        return int(_native.lib().qpm_engine_device_bytes(self.handle))

    def trace(self, first: int = 0, n: int | None = None) -> np.ndarray:
        done = ctypes.c_int64()
        _native.lib().qpm_engine_generation(self.handle, ctypes.byref(done))
        if n is None:
            n = done.value + 1 - first
        out = np.empty((n, 5), dtype=np.float64)
        _native.check(_native.lib().qpm_engine_read_trace(self.handle, first, n, out.ctypes.data),
                      "qpm_engine_read_trace")
        return out

    def best(self) -> Individual:
        """The final best individual (a column shard returns its columns [g0, g0 + Dl))."""
        genome = np.empty(self.Dl, dtype=np.float64)
        proj = np.empty(self.Dl, dtype=np.int8)
        fit = np.empty(1, dtype=np.float64)
        _native.check(_native.lib().qpm_engine_read_best(self.handle, genome.ctypes.data, proj.ctypes.data,
                                                         fit.ctypes.data), "qpm_engine_read_best")
        return Individual(genome=genome, projection=proj, fitness=float(fit[0]))

    def result(self, n_rows: int):
        """(trace rows [0, n_rows), best individual) with one copy and one synchronisation."""
        trace = np.empty((n_rows, 5), dtype=np.float64)
        genome = np.empty(self.Dl, dtype=np.float64)
        proj = np.empty(self.Dl, dtype=np.int8)
        fit = np.empty(1, dtype=np.float64)
        _native.check(_native.lib().qpm_engine_read_result(self.handle, 0, n_rows, trace.ctypes.data,
                                                           genome.ctypes.data, proj.ctypes.data, fit.ctypes.data),
                      "qpm_engine_read_result")
        return trace, Individual(genome=genome, projection=proj, fitness=float(fit[0]))

    def population(self):
        """(genome [NP, Dl], fitness [NP]); a column shard returns its columns."""
        genome = np.empty((self.NP, self.Dl), dtype=np.float64)
        fit = np.empty(self.NP, dtype=np.float64)
        _native.check(_native.lib().qpm_engine_read_population(self.handle, genome.ctypes.data, fit.ctypes.data),
                      "qpm_engine_read_population")
        return genome, fit


def _trace_rows(arr: np.ndarray) -> list:
    # tolist() hands back Python floats in one call (make_trace_row's types)
    return [(int(g), best, mean, f, sd) for g, best, mean, f, sd in arr.tolist()]


def _check_wolf_rates(sch: Schedules, generations: int) -> None:
    """The reference re-validates GWOParams with each generation's rates
    (replace(gwo, p_dist=..., p_sl=..., p_flip=...), optimizer.py:447-452) and
    so raises GWOParams' ValueError at the first generation whose scheduled
    rate leaves [0, 1]; the device takes the rates from a precomputed table, so
    the same check runs here, before generation 0, with the same message."""
    G = int(generations)
    if G < 1:
        return
    rest = 1.0 - np.arange(1, G + 1, dtype=np.float64) / float(G)  # the rates p0 (1 - g/G), g = 1..G
    for name, p0 in (("p_dist", sch.p_dist0), ("p_sl", sch.p_sl0), ("p_flip", sch.p_flip0)):
        v = p0 * rest
        bad = np.nonzero(~((v >= 0.0) & (v <= 1.0)))[0]
        if bad.size:  # the first failing generation, in GWOParams' field order at that generation
            g = int(bad[0]) + 1
            for nm, val in (("p_dist", sch.p_dist(g, G)), ("p_sl", sch.p_sl(g, G)), ("p_flip", sch.p_flip(g, G))):
                if not (0.0 <= val <= 1.0):
                    raise ValueError(f"{nm} must be in [0, 1], got {val}")


def _run(algorithm, objective, *, dimension, pop_size, generations, seed, de, gwo, sch, workers, bounds,
         fitness_mode, use_graph=True, chunk_size=None) -> RunResult:
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if chunk_size is not None and chunk_size < 1:  # parexec.BatchJob (parexec.py:69-70)
        raise ValueError(f"chunk_size must be >= 1, got {chunk_size}")
    if algorithm == "hybrid":
        _check_wolf_rates(sch, generations)
    if pop_size < 4:
        raise ValueError(f"population size must be >= 4, got {pop_size}")
    if dimension < 1:
        raise ValueError(f"dimension must be >= 1, got {dimension}")
    if dimension != getattr(objective, "dimension", dimension):
        raise ValueError(f"dimension {dimension} does not match the objective's {objective.dimension}")
    lo, hi = bounds
    if hi < lo:
        raise ValueError(f"bounds must satisfy min <= max, got ({lo}, {hi})")
    eng = Engine(objective, algorithm, pop_size=pop_size, generations=generations, seed=seed, de=de, gwo=gwo,
                 sch=sch, fitness_mode=fitness_mode, bounds=bounds)
    eng.init()
    eng.step(generations, use_graph=use_graph)
    eng.finalize()
    trace, best = eng.result(generations + 1)
    return RunResult(best=best, trace=_trace_rows(trace))


def run_hybrid(objective, *, dimension: int, pop_size: int, generations: int, seed: int,
               de_params: DEParams | None = None, gwo_params: GWOParams | None = None,
               schedules: Schedules | None = None, workers: int = 1, chunk_size: int | None = None,
               fitness_mode: str | None = None) -> RunResult:
    """DE -> select -> top-k -> discrete wolf update -> select -> F update, per generation."""
    de = replace(de_params) if de_params else DEParams()
    gwo = replace(gwo_params) if gwo_params else GWOParams()
    sch = replace(schedules) if schedules else Schedules()
    return _run("hybrid", objective, dimension=dimension, pop_size=pop_size, generations=generations, seed=seed,
                de=de, gwo=gwo, sch=sch, workers=workers, bounds=(de.x_min, de.x_max), fitness_mode=fitness_mode,
                chunk_size=chunk_size)


def run_de(objective, *, dimension: int, pop_size: int, generations: int, seed: int,
           de_params: DEParams | None = None, schedules: Schedules | None = None, workers: int = 1,
           chunk_size: int | None = None, fitness_mode: str | None = None) -> RunResult:
    de = replace(de_params) if de_params else DEParams()
    sch = replace(schedules) if schedules else Schedules()
    return _run("de", objective, dimension=dimension, pop_size=pop_size, generations=generations, seed=seed,
                de=de, gwo=GWOParams(), sch=sch, workers=workers, bounds=(de.x_min, de.x_max),
                fitness_mode=fitness_mode, chunk_size=chunk_size)


def run_gwo(objective, *, dimension: int, pop_size: int, generations: int, seed: int,
            gwo_params: GWOParams | None = None, workers: int = 1, chunk_size: int | None = None,
            bounds: tuple[float, float] = (-1.0, 1.0), fitness_mode: str | None = None) -> RunResult:
    gwo = replace(gwo_params) if gwo_params else GWOParams()
    return _run("gwo", objective, dimension=dimension, pop_size=pop_size, generations=generations, seed=seed,
                de=DEParams(), gwo=gwo, sch=Schedules(), workers=workers, bounds=bounds,
                fitness_mode=fitness_mode, chunk_size=chunk_size)


def run(algorithm: str, objective, *, dimension: int, pop_size: int, generations: int, seed: int,
        de_params: DEParams | None = None, gwo_params: GWOParams | None = None,
        schedules: Schedules | None = None, workers: int = 1, chunk_size: int | None = None,
        fitness_mode: str | None = None) -> RunResult:
    if algorithm == "hybrid":
        return run_hybrid(objective, dimension=dimension, pop_size=pop_size, generations=generations, seed=seed,
                          de_params=de_params, gwo_params=gwo_params, schedules=schedules, workers=workers,
                          chunk_size=chunk_size, fitness_mode=fitness_mode)
    if algorithm == "de":
        return run_de(objective, dimension=dimension, pop_size=pop_size, generations=generations, seed=seed,
                      de_params=de_params, schedules=schedules, workers=workers, chunk_size=chunk_size,
                      fitness_mode=fitness_mode)
    if algorithm == "gwo":
        return run_gwo(objective, dimension=dimension, pop_size=pop_size, generations=generations, seed=seed,
                       gwo_params=gwo_params, workers=workers, chunk_size=chunk_size, fitness_mode=fitness_mode)
    raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {algorithm!r}")
