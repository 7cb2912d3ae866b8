"""Host-side mirror of the reference API (CPU): validation, batch contracts with
plain callables, and the exported host helpers against reference fixtures.

The reference behaviour each test pins is cited inline
(/root/reference/pkg/src/qpmdesign/...).  Everything here runs without a GPU:
validation happens before the engine is created, and evaluate_batch with a
plain callable never touches the device.
"""

import numpy as np
import pytest

from conftest import golden
import paper_2511_01255_b200 as q
from paper_2511_01255_b200.parexec import BatchEvaluationError, BatchJob, evaluate_batch, reduce_best


def test_adaptive_f_update_matches_reference_fixtures():
    """adaptive_f_update (optimizer.py:277-299) bit-exact on the reference's own outputs."""
    fx = golden("operators.npz")
    for ci in fx["af_cases"]:
        g, tot, pstd, rng_, conv, base, adapt, decay = fx[f"af{ci}_args"]
        sch = q.Schedules(adaptive_branches=bool(adapt))
        st = q.AdaptiveState(generation=int(g), total_generations=int(tot), pop_std=pstd, fit_range=rng_,
                             convergence_rate=conv, decay_coeff=sch.decay_coeff(int(g), int(tot)), baseline_std=base)
        assert st.decay_coeff == decay
        assert q.adaptive_f_update(st, q.DEParams(), sch) == float(fx[f"af{ci}_f"])


def test_schedule_table_matches_adaptive_rule():
    """The device F envelope/decay columns equal the host rule's terms (optimizer.py:286-299)."""
    de, gwo, sch = q.DEParams(), q.GWOParams(), q.Schedules()
    tab = q.schedule_table(50, de, gwo, sch)
    for g in (0, 1, 17, 49, 50):
        st = q.AdaptiveState(generation=g, total_generations=50, pop_std=1.0, fit_range=10.0,
                             convergence_rate=1.0, decay_coeff=sch.decay_coeff(g, 50), baseline_std=1.0)
        nob = q.Schedules(adaptive_branches=False)
        f = q.adaptive_f_update(st, de, nob)
        assert f == min(max(tab[g, 0] * tab[g, 1], de.f_min), de.f_max)


def test_population_and_individual():
    """Population needs >= 4 individuals (optimizer.py:64-66); -0.0 projects to +1 (:52-56)."""
    ind = q.Individual.from_genome(np.array([-0.0, 0.0, -1e-300, 2.0]))
    assert list(ind.projection) == [1, 1, -1, 1]
    with pytest.raises(ValueError, match=">= 4"):
        q.Population([ind] * 3)
    pop = q.Population([q.Individual.from_genome(np.zeros(3), fitness=float(i)) for i in range(5)])
    assert pop.size == 5 and pop.dimension == 3
    assert np.array_equal(pop.fitness_values(), np.arange(5.0))
    with pytest.raises(ValueError, match="unevaluated"):
        q.Population([q.Individual.from_genome(np.zeros(3))] * 4).fitness_values()


class _Stub:
    """Stands in for an objective: validation raises before the engine (and the GPU) is touched."""

    dimension = 16


def _dummy_objective():
    return _Stub()


def test_chunk_size_validated_like_batchjob():
    """The reference raises BatchJob's ValueError for chunk_size < 1 (parexec.py:69-70)."""
    obj = _dummy_objective()
    for fn in (q.run_hybrid, q.run_de, q.run_gwo):
        with pytest.raises(ValueError, match="chunk_size must be >= 1, got 0"):
            fn(obj, dimension=16, pop_size=8, generations=2, seed=0, chunk_size=0)
    with pytest.raises(ValueError, match="chunk_size must be >= 1"):
        BatchJob(items=[1], chunk_size=0)
    with pytest.raises(ValueError, match="chunk_size must be >= 1"):
        reduce_best([1.0, 2.0], 1, chunk_size=-3)


def test_scheduled_wolf_rates_validated_like_reference():
    """run_hybrid re-validates GWOParams with each generation's rates (optimizer.py:447-452):
    out-of-range schedules raise GWOParams' message; G = 1 never reaches a rate != 0."""
    obj = _dummy_objective()
    with pytest.raises(ValueError, match=r"p_dist must be in \[0, 1\], got 1.35"):
        q.run_hybrid(obj, dimension=16, pop_size=8, generations=10, seed=0, schedules=q.Schedules(p_dist0=1.5))
    with pytest.raises(ValueError, match="p_sl must be in"):
        q.run_hybrid(obj, dimension=16, pop_size=8, generations=4, seed=0, schedules=q.Schedules(p_sl0=-0.1))
    with pytest.raises(ValueError, match="p_flip must be in"):
        q.run_hybrid(obj, dimension=16, pop_size=8, generations=4, seed=0,
                     schedules=q.Schedules(p_flip0=float("nan")))
    from paper_2511_01255_b200.optimizer import _check_wolf_rates

    _check_wolf_rates(q.Schedules(p_dist0=1.5), 1)  # p_dist(1, 1) = 0: valid, as in the reference
    _check_wolf_rates(q.Schedules(p_dist0=1.5), 0)


def test_evaluate_batch_plain_callables():
    """parexec contract with plain callables (test_parexec.py:53-72): order, item index, empty batch."""
    out = evaluate_batch(BatchJob(items=list(range(50)), workers=4, chunk_size=3), lambda x: float(x * x))
    assert np.array_equal(out, np.array([float(i * i) for i in range(50)]))

    def flaky(x):
        if x == 17:
            raise RuntimeError("boom")
        return float(x)

    with pytest.raises(BatchEvaluationError) as info:
        evaluate_batch(BatchJob(items=list(range(40)), workers=4, chunk_size=5), flaky)
    assert info.value.item_index == 17
    with pytest.raises(ValueError, match="non-empty"):
        BatchJob(items=[], workers=1)
    with pytest.raises(ValueError, match="workers"):
        evaluate_batch(BatchJob(items=[1], workers=0), float)


class _BlockObjective:
    """Any objective with evaluate_block takes the block path (parexec.py:88-92)."""

    def __init__(self):
        self.block_calls = 0

    def __call__(self, row):
        return float(np.sum(row))

    def evaluate_block(self, rows):
        self.block_calls += 1
        return np.sum(rows, axis=1).astype(np.float64)


class _FailingBlock(_BlockObjective):
    def __call__(self, row):
        if row[0] == 3:
            raise ValueError("bad row")
        return float(np.sum(row))

    def evaluate_block(self, rows):
        raise RuntimeError("block failed")


def test_evaluate_batch_block_path_any_objective():
    items = np.arange(40, dtype=np.int8).reshape(10, 4)
    obj = _BlockObjective()
    out = evaluate_batch(BatchJob(items=items, workers=3, chunk_size=2), obj)
    assert obj.block_calls == 1
    assert np.array_equal(out, items.sum(axis=1).astype(np.float64))
    bad = np.zeros((6, 4), dtype=np.int8)
    bad[4, 0] = 3
    with pytest.raises(BatchEvaluationError) as info:
        evaluate_batch(BatchJob(items=bad), _FailingBlock())
    assert info.value.item_index == 4


def test_reduce_best_host_validation():
    """parexec.reduce_best validation (parexec.py:133-137) and the device k bound (k <= 64)."""
    with pytest.raises(ValueError, match="empty"):
        reduce_best([], 1)
    with pytest.raises(ValueError, match="k must be"):
        reduce_best([1.0], 2)
    with pytest.raises(ValueError, match="k must be <= 64"):
        reduce_best(np.arange(100.0), 65)
    with pytest.raises(ValueError, match="workers"):
        reduce_best([1.0, 2.0], 1, workers=0)


def test_schedule_table_vectorised_equals_reference_expressions():
    """The per-generation scalars uploaded to the device are the reference's
    Python expressions (optimizer.py:157-171, 290, 563-564), bit for bit."""
    from paper_2511_01255_b200.optimizer import _schedule_table_reference, schedule_table

    for G in (0, 1, 2, 3, 7, 20, 999, 1000, 4097):
        for sch in (q.Schedules(), q.Schedules(phase_split=0.3, decay_strength=0.7, p_dist0=0.3, p_flip0=0.9)):
            for gwo in (q.GWOParams(), q.GWOParams(a=0.1, a_final=0.01)):
                de = q.DEParams(f_min=0.02, f_max=0.3, f=0.1)
                assert np.array_equal(schedule_table(G, de, gwo, sch), _schedule_table_reference(G, de, gwo, sch))
