"""Batched independent trials on one GPU or across a process group (drop-in for bench.run_trials /
compare_algorithms, /root/reference/pkg/src/qpmdesign/bench.py:91-159).

Trial t uses seed base_seed + t, exactly as the reference, and each trial is
the same device-resident run as `run_hybrid` / `run_de` / `run_gwo` (its
result is bit-identical to a lone run of that seed).  The trials run as a
population of runs: every trial owns an engine and a stream, all engines'
generation graphs are queued before any result is read, so small
configurations (C1: one generation is a few microseconds of GPU work) keep the
GPU busy with many runs at once.  The reference's RunConfig is replaced by
explicit keywords (config parsing is out of scope); `time_s` of a trial is its
batch's wall time divided by the batch size.

With group=<torch.distributed group> (one process per GPU) the seeds are dealt
round-robin over the ranks and the records all-gathered (all_gather_object,
host memory -- a few dozen floats per trial), so every rank returns exactly
the single-process result; there is no data-path collective because trials
are independent.
"""

import time
from dataclasses import dataclass, replace
from typing import Sequence

import numpy as np

from .optimizer import ALGORITHMS, DEParams, Engine, GWOParams, Schedules


@dataclass(frozen=True)
class RunStatistics:
    """One algorithm's aggregate over repeated trials (bench.py:24-39)."""

    algorithm: str
    trials: int
    average: float
    maximum: float
    minimum: float
    std: float
    mean_time_s: float
    mean_deff_norm: float

    def as_row(self) -> tuple:
        return (self.algorithm, self.average, self.maximum, self.minimum, self.std, self.mean_time_s,
                self.mean_deff_norm)


@dataclass(frozen=True)
class TrialRecord:
    trial: int
    seed: int
    final_fitness: float
    time_s: float
    deff_norm: float

    def as_row(self) -> tuple:
        return (self.trial, self.seed, self.final_fitness, self.time_s)


@dataclass(frozen=True)
class ComparisonReport:
    stats: dict
    mean_ratios: dict

    def ratio(self, numerator: str, denominator: str) -> float:
        return self.mean_ratios[f"{numerator}/{denominator}"]


def run_trials(objective, algorithm: str, trials: int, base_seed: int, *, dimension: int, pop_size: int,
               generations: int, de_params: DEParams | None = None, gwo_params: GWOParams | None = None,
               schedules: Schedules | None = None, fitness_mode: str | None = None,
               max_concurrent: int = 64, group=None) -> tuple[RunStatistics, list[TrialRecord]]:
    """Aggregate `trials` runs of one algorithm; trial t uses seed base_seed + t.

    group: a torch.distributed process group (one process per GPU) to spread
    the trials over -- rank r runs the trials t = r, r + W, r + 2W, ... on its
    own device and the records are all-gathered, so every rank returns the
    same statistics as a single-process run (the trials are independent; SURVEY
    §8(f) row 2: the paper's 30-seed protocol across 8 GPUs)."""
    if trials < 1:
        raise ValueError(f"trials must be >= 1, got {trials}")
    if algorithm not in ALGORITHMS:
        raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {algorithm!r}")
    if pop_size < 4:
        raise ValueError(f"population size must be >= 4, got {pop_size}")
    if dimension != objective.dimension:
        raise ValueError(f"dimension {dimension} does not match the objective's {objective.dimension}")
    if max_concurrent < 1:
        raise ValueError(f"max_concurrent must be >= 1, got {max_concurrent}")
    import torch

    de = replace(de_params) if de_params else DEParams()
    gwo = replace(gwo_params) if gwo_params else GWOParams()
    sch = replace(schedules) if schedules else Schedules()
    bounds = (de.x_min, de.x_max) if algorithm != "gwo" else (-1.0, 1.0)
    mine = list(range(trials))
    if group is not None:
        import torch.distributed as dist

        mine = mine[dist.get_rank(group)::dist.get_world_size(group)]
    records: list[TrialRecord] = []
    for first in range(0, len(mine), max_concurrent):
        batch = mine[first:first + max_concurrent]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        engines = [Engine(objective, algorithm, pop_size=pop_size, generations=generations, seed=base_seed + t,
                          de=de, gwo=gwo, sch=sch, fitness_mode=fitness_mode, bounds=bounds) for t in batch]
        for eng in engines:  # queue every run before reading any result
            eng.init()
            eng.step(generations)
            eng.finalize()
        bests = [eng.best() for eng in engines]
        torch.cuda.synchronize()
        per_trial = (time.perf_counter() - t0) / len(batch)
        del engines
        for t, best in zip(batch, bests):
            deff = float(np.mean(objective.normalized_gains(best.projection)))
            records.append(TrialRecord(trial=t, seed=base_seed + t, final_fitness=best.fitness, time_s=per_trial,
                                       deff_norm=deff))
    if group is not None:
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, records, group=group)
        records = sorted((r for part in parts for r in part), key=lambda r: r.trial)
    return _statistics(algorithm, records), records


def _statistics(algorithm: str, records: list) -> RunStatistics:
    """bench.run_trials' aggregate (bench.py:133-146) of records in trial order."""
    finals = np.array([r.final_fitness for r in records])
    n = len(records)
    return RunStatistics(
        algorithm=algorithm,
        trials=n,
        average=float(np.mean(finals)),
        maximum=float(np.max(finals)),
        minimum=float(np.min(finals)),
        std=float(np.std(finals, ddof=1)) if n > 1 else 0.0,
        mean_time_s=float(np.mean([r.time_s for r in records])),
        mean_deff_norm=float(np.mean([r.deff_norm for r in records])),
    )


def compare_algorithms(objective, trials: int, base_seed: int, algorithms: Sequence[str] = ALGORITHMS,
                       **kwargs) -> ComparisonReport:
    """Seed-matched comparison with every pairwise ratio of means (bench.py:141-159)."""
    if trials < 10:
        raise ValueError(f"algorithm comparisons need trials >= 10, got {trials}")
    stats = {}
    for algorithm in algorithms:
        result, _ = run_trials(objective, algorithm, trials, base_seed, **kwargs)
        stats[result.algorithm] = result
    ratios = {}
    for a in stats:
        for b in stats:
            if a != b and stats[b].average != 0.0:
                ratios[f"{a}/{b}"] = stats[a].average / stats[b].average
    return ComparisonReport(stats=stats, mean_ratios=ratios)
