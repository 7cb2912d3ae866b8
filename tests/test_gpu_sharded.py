"""GPU: the column-sharded (multi-GPU) engine path, emulated with W shard
engines on one GPU (EmulatedShards), must reproduce the single-engine run bit
for bit (fast mode: the shards scan the single-GPU fitness segments and every
shard stitches all of them in the single-GPU order).

Each shard runs exactly the kernels a real rank runs (per-gene kernels on its
columns of all rows, segment scans, the replicated finish / selection /
statistics); only the NCCL all-gather of the segment partials is replaced by
device copies.  A 1-rank NCCL communicator runs the real collective path.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import torch

    torch.cuda.set_device(0)
    import paper_2511_01255_b200 as pkg

    return pkg


def _kw(q, algorithm, NP=48, G=25, seed=11):
    gwo = q.GWOParams(a=0.1, a_final=0.01) if algorithm == "gwo" else q.GWOParams()
    return dict(pop_size=NP, generations=G, seed=seed, de=q.DEParams(), gwo=gwo, sch=q.Schedules())


@pytest.mark.parametrize("algorithm", ["hybrid", "de", "gwo"])
@pytest.mark.parametrize("world,D", [(2, 3000), (3, 5000), (4, 5000), (8, 10_000)])
def test_emulated_shards_match_single_engine(q, algorithm, world, D):
    from paper_2511_01255_b200.distributed import EmulatedShards, shard_columns

    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, D, mode="fast")
    kw = _kw(q, algorithm)
    single = q.Engine(obj, algorithm, **kw)
    single.init()
    single.step(kw["generations"])
    single.finalize()
    want = single.trace()
    shards = EmulatedShards(obj, algorithm, world, **kw)
    for r, e in enumerate(shards.engines):
        assert (e.g0, e.g0 + e.Dl) == shard_columns(D, world, r)
    shards.init()
    shards.step(kw["generations"])
    shards.finalize()
    for e in shards.engines:
        assert np.array_equal(e.trace(), want)
    g_single, f_single = single.population()
    g_shard, f_shard = shards.population()
    assert np.array_equal(g_shard, g_single)
    assert np.array_equal(f_shard, f_single)
    b, bs = shards.best(), single.best()
    assert b.fitness == bs.fitness
    assert np.array_equal(b.genome, bs.genome) and np.array_equal(b.projection, bs.projection)


def test_emulated_shards_multi_wavelength(q):
    """Several pump wavelengths (gains per wavelength, multi objective) through the sharded finish."""
    from paper_2511_01255_b200.distributed import EmulatedShards

    pumps = tuple(float(w) for w in np.linspace(1390.0, 1420.0, 3))
    obj = q.make_objective(q.ObjectiveSpec("multi_thg", pumps), q.default_dispersion(), 0.5, 9000, mode="fast")
    kw = _kw(q, "hybrid", NP=32, G=12)
    single = q.Engine(obj, "hybrid", **kw)
    single.init()
    single.step(kw["generations"])
    shards = EmulatedShards(obj, "hybrid", 2, **kw)
    shards.init()
    shards.step(kw["generations"])
    for e in shards.engines:
        assert np.array_equal(e.trace(), single.trace())


def test_sharded_engine_rejects_bad_shards(q):
    from paper_2511_01255_b200 import _native
    from paper_2511_01255_b200.distributed import ShardedEngine

    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 64)
    kw = _kw(q, "hybrid", NP=12, G=3)
    with pytest.raises(ValueError, match="outside"):
        ShardedEngine.create(obj, "hybrid", rank=3, world=3, **kw)
    with pytest.raises(_native.QpmError, match="segments"):  # D = 64: one fitness segment
        ShardedEngine.create(obj, "hybrid", rank=0, world=2, **kw)
    big = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 3000,
                           mode="exact")
    with pytest.raises(_native.QpmError, match="fast mode"):
        ShardedEngine.create(big, "hybrid", rank=0, world=2, **kw)
    fast = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 3000)
    eng = ShardedEngine.create(fast, "hybrid", rank=1, world=2, **kw)
    eng.init()  # emulated shard: stops after the generation-0 scan
    with pytest.raises(_native.QpmError, match="before qpm_engine_init"):
        eng.step(1)
    eng.init_finish()  # (without the other rank's partials: only the state machine is exercised)
    with pytest.raises(_native.QpmError, match="communicator"):
        eng.step(1)
    with pytest.raises(_native.QpmError, match="pending"):
        eng.init_finish()


@pytest.mark.parametrize("algorithm", ["hybrid", "de", "gwo"])
def test_one_rank_nccl_communicator_in_graph(q, algorithm):
    """With a 1-rank communicator the engine takes the multi-GPU path for real
    (segment scan, ncclAllGather captured in the generation graph, replicated
    finish): the trace must equal the single-GPU engine's."""
    from paper_2511_01255_b200.distributed import ShardedEngine, nccl_unique_id

    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 2500)
    kw = _kw(q, algorithm, NP=32, G=12, seed=4)
    ref = q.Engine(obj, algorithm, **kw)
    ref.init()
    ref.step(12)
    eng = ShardedEngine.create(obj, algorithm, rank=0, world=1, nccl_id=nccl_unique_id(), **kw)
    eng.init()
    eng.prepare(12)  # the allgather captured in the generation graphs
    eng.step(12, use_graph=True)
    assert np.array_equal(eng.trace(), ref.trace())
