"""GPU: checkpoint / resume of a device run (qpm_engine_checkpoint / _restore).

A run stopped after k generations, checkpointed to host bytes, and resumed in
a new engine created with the same arguments must be bit-identical to the
uninterrupted run: every trace row, the population and the final best
(a checkpoint is (g, F, window, baseline std, genome, fitness,
best_prev); the counter RNG has no state).
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


def _engine(q, obj, algorithm, G, seed):
    gwo = q.GWOParams(a=0.1, a_final=0.01) if algorithm == "gwo" else q.GWOParams()
    return q.Engine(obj, algorithm, pop_size=64, generations=G, seed=seed, de=q.DEParams(), gwo=gwo,
                    sch=q.Schedules())


@pytest.mark.parametrize("algorithm", ["hybrid", "de", "gwo"])
@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_resume_is_bit_identical(q, algorithm, mode):
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 2000, mode=mode)
    G, k = 40, 17
    ref = _engine(q, obj, algorithm, G, 5)
    ref.init()
    ref.step(G)
    ref.finalize()
    want_trace, want_pop, want_best = ref.trace(), ref.population(), ref.best()

    a = _engine(q, obj, algorithm, G, 5)
    a.init()
    a.prepare(k)
    a.step(k)  # graph replays before the checkpoint
    data = a.checkpoint()
    assert np.array_equal(a.trace(), want_trace[:k + 1])
    del a

    b = _engine(q, obj, algorithm, G, 5)
    b.restore(data)
    assert np.array_equal(b.trace(), want_trace[:k + 1])
    b.step(G - k, use_graph=False)
    b.finalize()
    assert np.array_equal(b.trace(), want_trace)
    g, f = b.population()
    assert np.array_equal(g, want_pop[0]) and np.array_equal(f, want_pop[1])
    best = b.best()
    assert best.fitness == want_best.fitness
    assert np.array_equal(best.genome, want_best.genome) and np.array_equal(best.projection, want_best.projection)


def test_restore_rejects_a_different_run(q):
    from paper_2511_01255_b200._native import QpmError

    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 500)
    a = _engine(q, obj, "hybrid", 10, 1)
    a.init()
    a.step(3)
    data = a.checkpoint()
    other = _engine(q, obj, "hybrid", 10, 2)  # another seed
    with pytest.raises(QpmError, match="different run"):
        other.restore(data)
    used = _engine(q, obj, "hybrid", 10, 1)
    used.init()
    with pytest.raises(QpmError, match="freshly created"):
        used.restore(data)
    with pytest.raises(QpmError, match="not a qpm engine checkpoint"):
        _engine(q, obj, "hybrid", 10, 1).restore(b"\0" * len(data))
