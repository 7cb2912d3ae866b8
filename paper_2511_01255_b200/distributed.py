"""Multi-GPU HWSDA: one process per GPU, rows sharded, NCCL over NVLink.

Scheme ("exact scheme"):

* every rank keeps the whole population (C3: 6.5 GB of f64 genome, far below
  180 GB of HBM) and owns an equal contiguous slice of rows;
* per generation each rank builds and scores the DE trials of its own rows,
  then the candidate fitness vector (NP doubles) is all-gathered; every rank
  recomputes the trials other ranks accepted from the same counter streams
  (bit-identical arithmetic), so the replicas stay identical without moving
  genomes;
* the wolf phase scores own rows, then all-gathers the candidate fitness and
  the candidates' sign bits (D/8 bytes per row), which is cheaper than
  recomputing three random draws per gene;
* leaders, selection, statistics and the F update are computed redundantly
  on every rank from identical data, so they need no further collective.

The collectives run inside the engine (libqpm_b200.so calls ncclAllGather on
the engine stream, captured into the per-generation CUDA graph).  The NCCL
communicator is bootstrapped from a unique id that rank 0 creates and
torch.distributed broadcasts.  `EmulatedShards` drives W shard engines on one
GPU with host-side exchanges between phases, so the sharded path can be
tested bit-exactly against the single engine without several GPUs.
"""

import ctypes
from dataclasses import replace

import numpy as np

from . import _native
from .optimizer import DEParams, Engine, GWOParams, RunResult, Schedules, _trace_rows


def shard_rows(pop_size: int, world: int, rank: int) -> tuple[int, int]:
    """Equal contiguous row slice of `rank` (NP must be a multiple of world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    if pop_size % world:
        raise ValueError(f"population size {pop_size} is not a multiple of the rank count {world}")
    per = pop_size // world
    return rank * per, (rank + 1) * per


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _native.check(_native.lib().qpm_nccl_unique_id(buf), "qpm_nccl_unique_id")
    return bytes(buf)


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0's NCCL id on every rank (torch.distributed object broadcast)."""
    import torch.distributed as dist

    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class ShardedEngine(Engine):
    """An Engine owning rows [lo, hi) of a run spread over `world` ranks."""

    @classmethod
    def create(cls, objective, algorithm, *, pop_size, generations, seed, de, gwo, sch, rank, world,
               nccl_id=None, fitness_mode=None, bounds=(-1.0, 1.0), stream=None):
        eng = Engine.__new__(cls)
        eng.rank, eng.world = rank, world
        eng.row_lo, eng.row_hi = shard_rows(pop_size, world, rank)
        Engine.__init__(eng, objective, algorithm, pop_size=pop_size, generations=generations, seed=seed, de=de,
                        gwo=gwo, sch=sch, fitness_mode=fitness_mode, bounds=bounds, stream=stream,
                        row_range=(eng.row_lo, eng.row_hi))
        if nccl_id is not None:
            idb = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
            _native.check(_native.lib().qpm_engine_set_comm(eng.handle, rank, world, idb), "qpm_engine_set_comm")
        elif world > 1:
            _native.check(_native.lib().qpm_engine_set_shard(eng.handle, rank, world), "qpm_engine_set_shard")
        return eng

    @property
    def phases(self) -> int:
        return int(_native.lib().qpm_engine_phases(self.handle))

    def run_phase(self, phase: int):
        _native.check(_native.lib().qpm_engine_run_phase(self.handle, int(phase)), "qpm_engine_run_phase")

    def exchange_from(self, other: "ShardedEngine", phase: int):
        _native.check(_native.lib().qpm_engine_exchange_from(self.handle, other.handle, int(phase)),
                      "qpm_engine_exchange_from")


class EmulatedShards:
    """W shard engines of one run on one GPU, exchanging between phases.

    Test harness for the sharded protocol: every kernel a real rank runs is
    run by its shard engine; the NCCL all-gather is replaced by device copies
    of each shard's own slices into the other shards' buffers.
    """

    def __init__(self, objective, algorithm, world: int, **kw):
        self.engines = [ShardedEngine.create(objective, algorithm, rank=r, world=world, nccl_id=None, **kw)
                        for r in range(world)]

    def init(self):
        for e in self.engines:
            e.init()

    def step(self, n: int):
        import torch

        phases = self.engines[0].phases
        for _ in range(n):
            for ph in range(phases):
                if ph > 0:
                    torch.cuda.synchronize()
                    for dst in self.engines:
                        for src in self.engines:
                            if src is not dst:
                                dst.exchange_from(src, ph)
                for e in self.engines:
                    e.run_phase(ph)
        torch.cuda.synchronize()

    def finalize(self):
        for e in self.engines:
            e.finalize()


def run_sharded(algorithm: str, objective, *, dimension: int, pop_size: int, generations: int, seed: int,
                de_params: DEParams | None = None, gwo_params: GWOParams | None = None,
                schedules: Schedules | None = None, fitness_mode: str | None = None, group=None,
                use_graph: bool = True) -> RunResult:
    """The run on all ranks of `group` (torch.distributed, NCCL); every rank returns the same result."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    de = replace(de_params) if de_params else DEParams()
    gwo = replace(gwo_params) if gwo_params else GWOParams()
    sch = replace(schedules) if schedules else Schedules()
    if dimension != objective.dimension:
        raise ValueError(f"dimension {dimension} does not match the objective's {objective.dimension}")
    uid = broadcast_unique_id(group) if world > 1 else None
    bounds = (de.x_min, de.x_max) if algorithm != "gwo" else (-1.0, 1.0)
    eng = ShardedEngine.create(objective, algorithm, pop_size=pop_size, generations=generations, seed=seed, de=de,
                               gwo=gwo, sch=sch, rank=rank, world=world, nccl_id=uid, fitness_mode=fitness_mode,
                               bounds=bounds)
    eng.init()
    eng.step(generations, use_graph=use_graph)
    eng.finalize()
    return RunResult(best=eng.best(), trace=_trace_rows(eng.trace(0, generations + 1)))


def replicas_trace_equal(traces) -> bool:
    first = np.asarray(traces[0])
    return all(np.array_equal(first, np.asarray(t)) for t in traces[1:])
