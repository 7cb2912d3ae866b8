"""GPU: the sharded (multi-GPU) engine path, emulated with W shard engines on
one GPU (EmulatedShards), must reproduce the single-engine trace bit for bit.

Each shard runs exactly the kernels a real rank runs (own-row trials, own-row
fitness, recompute of foreign accepted trials, commit of all-gathered wolf
candidates); only the NCCL all-gather is replaced by device copies.
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


@pytest.mark.parametrize("algorithm", ["hybrid", "de", "gwo"])
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_emulated_shards_match_single_engine(q, algorithm, world, mode):
    from paper_2511_01255_b200.distributed import EmulatedShards

    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, 700, mode=mode)
    NP, G = 48, 25
    gwo = q.GWOParams(a=0.1, a_final=0.01) if algorithm == "gwo" else q.GWOParams()
    kw = dict(pop_size=NP, generations=G, seed=11, de=q.DEParams(), gwo=gwo, sch=q.Schedules())
    single = q.Engine(obj, algorithm, **kw)
    single.init()
    single.step(G)
    single.finalize()
    want = single.trace()
    shards = EmulatedShards(obj, algorithm, world, **kw)
    shards.init()
    shards.step(G)
    shards.finalize()
    for e in shards.engines:
        assert np.array_equal(e.trace(), want)
        assert np.array_equal(e.population()[0], single.population()[0])
    assert shards.engines[-1].best().fitness == single.best().fitness


def test_sharded_engine_rejects_bad_shards(q):
    from paper_2511_01255_b200 import _native
    from paper_2511_01255_b200.distributed import ShardedEngine

    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 64)
    kw = dict(pop_size=12, generations=3, seed=1, de=q.DEParams(), gwo=q.GWOParams(), sch=q.Schedules())
    with pytest.raises(ValueError, match="multiple"):
        ShardedEngine.create(obj, "hybrid", rank=0, world=5, **kw)
    eng = ShardedEngine.create(obj, "hybrid", rank=1, world=3, **kw)
    eng.init()
    with pytest.raises(_native.QpmError, match="communicator"):
        eng.step(1)


def test_one_rank_nccl_communicator_in_graph(q):
    """The NCCL all-gathers are captured into the generation graph; with a
    1-rank communicator they run for real and must not change the trace."""
    from paper_2511_01255_b200.distributed import ShardedEngine, nccl_unique_id

    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 500)
    kw = dict(pop_size=32, generations=12, seed=4, de=q.DEParams(), gwo=q.GWOParams(), sch=q.Schedules())
    ref = q.Engine(obj, "hybrid", **kw)
    ref.init()
    ref.step(12)
    eng = ShardedEngine.create(obj, "hybrid", rank=0, world=1, nccl_id=nccl_unique_id(), **kw)
    eng.init()
    eng.step(12, use_graph=True)
    assert np.array_equal(eng.trace(), ref.trace())


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_engines_sharing_a_problem_run_concurrently(q, mode):
    """Engines built on one objective own their fitness scratch: stepped
    concurrently on their own streams they reproduce their solo traces."""
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 900, mode=mode)
    kws = [dict(pop_size=64, generations=30, seed=s, de=q.DEParams(), gwo=q.GWOParams(), sch=q.Schedules())
           for s in (1, 2, 3)]
    solo = []
    for kw in kws:
        e = q.Engine(obj, "hybrid", **kw)
        e.init()
        e.step(30)
        solo.append(e.trace())
    engines = [q.Engine(obj, "hybrid", **kw) for kw in kws]
    for e in engines:
        e.init()
    for _ in range(30):
        for e in engines:
            e.step(1)
    for e, want in zip(engines, solo):
        assert np.array_equal(e.trace(), want)
