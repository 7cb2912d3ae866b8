"""Multi-GPU HWSDA: one process per GPU, genes sharded by columns, NCCL over NVLink.

Scheme (a column variant of SURVEY.md §8(e)'s exact scheme):

* the genes are split into contiguous column ranges aligned to the fitness
  segments: rank k owns the genes under segments [floor(k S / W),
  floor((k+1) S / W)) of every individual (S = the problem's segments);
* every per-gene operation only touches its own column of other rows: the DE
  trial x_r1 + F (x_r2 - x_r3) and the crossover mask, the wolf draws and the
  leader vote (leaders' columns are local), init_population, run_gwo's
  continuous move; so each rank runs them on its columns of all NP rows, with
  the stream positions of the global gene index (bit-identical draws);
* each rank scans the fitness segments of its columns for all rows and
  pre-stitches them into its stitch super-blocks (the fixed single-GPU tree:
  min(8, S) contiguous super-blocks); those partials (NP x 48 B per owned
  super-block, about NP x 8 x 48 B over all ranks) are all-gathered and every
  rank finishes and scores all rows (fast-mode fitness bit-identical to one
  GPU);
* selection, leaders, statistics and the F update run replicated on every
  rank from identical data, so they need no further collective.

Per generation a hybrid run all-gathers the partials twice (DE and wolf
candidates), 393 KB each at NP 1024 / 3.1 MB at NP 8192 (one wavelength);
nothing else moves: no genome rows, no recomputation.  The
collectives run inside the engine (libqpm_b200.so calls ncclAllGather on the
engine stream, captured into the per-generation CUDA graph).  The NCCL
communicator is bootstrapped from a unique id that rank 0 creates and
torch.distributed broadcasts.  `EmulatedShards` drives W shard engines on one
GPU with device-copy exchanges between phases, so the sharded path is tested
bit-exactly against the single engine without several GPUs.
"""

import ctypes
from dataclasses import replace

import numpy as np

from . import _native
from .optimizer import DEParams, Engine, GWOParams, Individual, RunResult, Schedules, _trace_rows


def shard_columns(D: int, world: int, rank: int, n_wl: int = 1, seg_chunks: int | None = None) -> tuple[int, int]:
    """Gene columns [g0, g1) of `rank` (the engine's split, qpm_engine_create):
    the problem's S fitness segments (seg_chunks 128-domain chunks each; by
    default 3 for one wavelength, 2 when that leaves fewer than 16 segments,
    4 min(n_wl, 8) with several) form B = min(8, S) stitch super-blocks,
    super-block b = segments [floor(b S / B), floor((b+1) S / B)); rank k owns
    super-blocks [floor(k B / W), floor((k+1) B / W)) and the genes under them."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    words = -(-(-(-D // 32)) // 4) * 4
    nchunks = words // 4
    if seg_chunks is None:  # qpm_problem_create's default
        seg_chunks = 4 * min(n_wl, 8) if n_wl > 1 else (2 if -(-nchunks // 3) < 16 else 3)
    seg_chunks = max(1, min(nchunks, seg_chunks))
    S = -(-nchunks // seg_chunks)
    B = min(8, S)
    if B < world:
        raise ValueError(f"{S} fitness segments ({B} stitch super-blocks) cannot be split over {world} ranks")
    sb0, sb1 = rank * B // world, (rank + 1) * B // world
    lo, hi = sb0 * S // B, sb1 * S // B
    seg = seg_chunks * 128
    return lo * seg, min(D, hi * seg)


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
    """An Engine owning the gene columns [g0, g0 + Dl) of a run spread over `world` ranks."""

    @classmethod
    def create(cls, objective, algorithm, *, pop_size, generations, seed, de, gwo, sch, rank, world,
               nccl_id=None, fitness_mode=None, bounds=(-1.0, 1.0), stream=None):
        if world < 1 or not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside [0, {world})")
        eng = Engine.__new__(cls)
        eng.rank, eng.world = rank, world
        Engine.__init__(eng, objective, algorithm, pop_size=pop_size, generations=generations, seed=seed, de=de,
                        gwo=gwo, sch=sch, fitness_mode=fitness_mode, bounds=bounds, stream=stream,
                        shard=(rank, world))
        eng.emulated = nccl_id is None and world > 1
        if nccl_id is not None:
            idb = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
            _native.check(_native.lib().qpm_engine_set_comm(eng.handle, rank, world, idb), "qpm_engine_set_comm")
        return eng

    @property
    def phases(self) -> int:
        return int(_native.lib().qpm_engine_phases(self.handle))

    def run_phase(self, phase: int):
        _native.check(_native.lib().qpm_engine_run_phase(self.handle, int(phase)), "qpm_engine_run_phase")

    def init_finish(self):
        _native.check(_native.lib().qpm_engine_init_finish(self.handle), "qpm_engine_init_finish")

    def exchange_from(self, other: "ShardedEngine", phase: int):
        _native.check(_native.lib().qpm_engine_exchange_from(self.handle, other.handle, int(phase)),
                      "qpm_engine_exchange_from")

    def wait(self, timeout_s: float | None = None):
        """Block until the queued generations finish, with failure detection
        (qpm_engine_wait): an NCCL asynchronous error, or no completion within
        timeout_s, aborts the communicator and raises QpmError."""
        ms = -1 if timeout_s is None else int(timeout_s * 1e3)
        _native.check(_native.lib().qpm_engine_wait(self.handle, ms), "qpm_engine_wait")

    def partials_slot(self) -> int:
        n = ctypes.c_int64()
        _native.check(_native.lib().qpm_engine_partials_info(self.handle, ctypes.byref(n), None, None),
                      "qpm_engine_partials_info")
        return int(n.value)

    def partials_read(self) -> np.ndarray:
        out = np.empty(self.partials_slot(), dtype=np.float64)
        _native.check(_native.lib().qpm_engine_partials_read(self.handle, out.ctypes.data), "qpm_engine_partials_read")
        return out

    def partials_write(self, rank: int, slot: np.ndarray):
        slot = np.ascontiguousarray(slot, dtype=np.float64)
        if slot.size != self.partials_slot():
            raise ValueError(f"slot has {slot.size} doubles, the engine's is {self.partials_slot()}")
        _native.check(_native.lib().qpm_engine_partials_write(self.handle, int(rank), slot.ctypes.data),
                      "qpm_engine_partials_write")

    def best_columns(self) -> tuple[int, Individual]:
        """(g0, this shard's columns of the final best individual)."""
        return self.g0, Engine.best(self)


def assemble_best(parts, D: int) -> Individual:
    """The full best individual from every rank's (g0, columns) part."""
    genome = np.empty(D, dtype=np.float64)
    proj = np.empty(D, dtype=np.int8)
    fit = None
    for g0, ind in parts:
        genome[g0:g0 + ind.genome.size] = ind.genome
        proj[g0:g0 + ind.projection.size] = ind.projection
        fit = ind.fitness
    return Individual(genome=genome, projection=proj, fitness=fit)


class EmulatedShards:
    """W shard engines of one run on one GPU, exchanging between phases.

    Test harness for the sharded protocol: every kernel a real rank runs is
    run by its shard engine; the NCCL all-gather is replaced by device copies
    of each shard's super-block partials into the other shards' buffers.
    """

    def __init__(self, objective, algorithm, world: int, **kw):
        self.D = objective.dimension
        self.engines = [ShardedEngine.create(objective, algorithm, rank=r, world=world, nccl_id=None, **kw)
                        for r in range(world)]

    def _exchange(self, ph):
        import torch

        torch.cuda.synchronize()
        for dst in self.engines:
            for src in self.engines:
                if src is not dst:
                    dst.exchange_from(src, ph)

    def init(self):
        for e in self.engines:
            e.init()
        self._exchange(0)
        for e in self.engines:
            e.init_finish()

    def step(self, n: int):
        import torch

        phases = self.engines[0].phases
        for _ in range(n):
            for ph in range(phases):
                if ph > 0:
                    self._exchange(ph)
                for e in self.engines:
                    e.run_phase(ph)
        torch.cuda.synchronize()

    def finalize(self):
        for e in self.engines:
            e.finalize()

    def best(self) -> Individual:
        return assemble_best([e.best_columns() for e in self.engines], self.D)

    def population(self):
        """(genome [NP, D], fitness [NP]) assembled from the shards' columns."""
        parts = [(e.g0, e.population()) for e in self.engines]
        NP = self.engines[0].NP
        genome = np.empty((NP, self.D), dtype=np.float64)
        for g0, (g, _) in parts:
            genome[:, g0:g0 + g.shape[1]] = g
        return genome, parts[0][1][1]


class HostExchangeShard:
    """This process's shard engine of a column-sharded run whose exchanges
    go through host memory and a torch.distributed group of any backend
    (gloo on CPU) instead of the in-graph ncclAllGather.

    The kernels are the real shard engine's; only the transport differs: after
    each phase the rank's partial slot is read to the host, all-gathered over
    the group and the peers' slots written back (qpm_engine_partials_*).  It
    is how the sharded protocol is exercised across a process boundary on a
    single GPU (NCCL cannot place two ranks on one device), and a slow but
    working path for hosts without NCCL peers.
    """

    def __init__(self, objective, algorithm, *, group=None, **kw):
        import torch.distributed as dist

        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.engine = ShardedEngine.create(objective, algorithm, rank=self.rank, world=self.world, nccl_id=None,
                                           **kw)
        self.D = objective.dimension
        self.exchanged_bytes = 0

    def _exchange(self):
        import torch
        import torch.distributed as dist

        mine = torch.from_numpy(self.engine.partials_read())
        parts = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(parts, mine, group=self.group)
        for r, p in enumerate(parts):
            if r != self.rank:
                self.engine.partials_write(r, p.numpy())
        self.exchanged_bytes += mine.numel() * 8 * self.world

    def init(self):
        self.engine.init()
        self._exchange()
        self.engine.init_finish()

    def step(self, n: int):
        for _ in range(n):
            for ph in range(self.engine.phases):
                if ph > 0:
                    self._exchange()
                self.engine.run_phase(ph)

    def finalize(self):
        self.engine.finalize()

    def trace(self):
        return self.engine.trace()

    def best(self) -> Individual:
        import torch.distributed as dist

        parts = [None] * self.world
        dist.all_gather_object(parts, self.engine.best_columns(), group=self.group)
        return assemble_best(parts, self.D)


def run_sharded(algorithm: str, objective, *, dimension: int, pop_size: int, generations: int, seed: int,
                de_params: DEParams | None = None, gwo_params: GWOParams | None = None,
                schedules: Schedules | None = None, fitness_mode: str | None = None, group=None,
                use_graph: bool = True, timeout_s: float | None = 600.0) -> RunResult:
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
    eng.wait(timeout_s)  # failure detection: a dead or stuck peer raises instead of hanging
    part = eng.best_columns()
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, part, group=group)
    else:
        parts = [part]
    return RunResult(best=assemble_best(parts, dimension), trace=_trace_rows(eng.trace(0, generations + 1)))


def replicas_trace_equal(traces) -> bool:
    first = np.asarray(traces[0])
    return all(np.array_equal(first, np.asarray(t)) for t in traces[1:])
