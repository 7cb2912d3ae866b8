"""the exhaustive oracle (bench.brute_force_oracle)
and batched independent trials (bench.run_trials / compare_algorithms).

CPU tests pin the oracle restatement of the exhaustive search against the
reference's own brute_force_oracle results (tests/golden/search.npz); GPU
tests run the device search (qpm_brute_force) and the population-of-runs
trial batch through the package API.
"""

import json

import numpy as np
import pytest

from conftest import golden, spec_of
from oracle import oracle as O
from test_oracle_golden import problem_from_spec

SEARCH_NAMES = json.loads(str(golden("search.npz")["names"]))


def lex_patterns(n):
    idx = np.arange(1 << n, dtype=np.int64)
    return (1 - 2 * ((idx[:, None] >> np.arange(n - 1, -1, -1)) & 1)).astype(np.int8)


@pytest.mark.parametrize("name", SEARCH_NAMES)
def test_oracle_exhaustive_search_matches_reference(name):
    fx = golden("search.npz")
    spec = spec_of(fx, name)
    n = spec["count"]
    vals = O.evaluate_block(problem_from_spec(spec), lex_patterns(n))
    best = int(np.argmax(vals))  # first maximum: the lexicographic tie-break
    assert best == int(fx[f"{name}__index"])
    assert vals[best] == float(fx[f"{name}__fit"])


def test_lexicographic_signs_order():
    from paper_2511_01255_b200.search import lexicographic_signs

    assert lexicographic_signs(0, 4).tolist() == [1, 1, 1, 1]
    assert lexicographic_signs(1, 4).tolist() == [1, 1, 1, -1]
    assert lexicographic_signs(8, 4).tolist() == [-1, 1, 1, 1]
    assert np.array_equal(np.stack([lexicographic_signs(i, 5) for i in range(32)]), lex_patterns(5))


def test_search_and_trials_validation():
    import paper_2511_01255_b200 as q

    class Dummy:
        dimension = 5
        mode = "fast"

    with pytest.raises(ValueError, match="n must be >= 1"):
        q.brute_force_oracle(Dummy(), 0)
    with pytest.raises(ValueError, match="refuses n > 20"):
        q.brute_force_oracle(Dummy(), 21)
    with pytest.raises(ValueError, match="does not match"):
        q.brute_force_oracle(Dummy(), 4)
    with pytest.raises(ValueError, match="trials must be >= 1"):
        q.run_trials(Dummy(), "hybrid", 0, 0, dimension=5, pop_size=8, generations=1)
    with pytest.raises(ValueError, match="algorithm must be one of"):
        q.run_trials(Dummy(), "pso", 2, 0, dimension=5, pop_size=8, generations=1)
    with pytest.raises(ValueError, match="trials >= 10"):
        q.compare_algorithms(Dummy(), 9, 0, dimension=5, pop_size=8, generations=1)


# ------------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def q():
    import torch

    torch.cuda.set_device(0)
    import paper_2511_01255_b200 as pkg

    return pkg


def objective_for(q, spec, mode):
    prov = q.MismatchTable({float(w): q.PhaseMismatchPair(*dk) for w, dk in zip(spec["pumps"], spec["dks"])})
    s = q.ObjectiveSpec(spec["variant"], tuple(spec["pumps"]), g0=spec["g0"], beta=spec["beta"],
                        normalization=spec["normalization"])
    return q.make_objective(s, prov, spec["thickness"], spec["count"], mode=mode)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SEARCH_NAMES)
def test_device_search_matches_reference(q, name):
    fx = golden("search.npz")
    spec = spec_of(fx, name)
    n = spec["count"]
    want_i, want_f = int(fx[f"{name}__index"]), float(fx[f"{name}__fit"])
    signs, fit = q.brute_force_oracle(objective_for(q, spec, "exact"), n, chunk=777)  # ragged chunks
    assert np.array_equal(signs, q.lexicographic_signs(want_i, n))
    assert fit == want_f  # exact mode: bit-identical
    # fast mode: an optimum up to rounding (patterns that tie exactly in the
    # reference arithmetic, e.g. mirror images, may resolve either way)
    signs, fit = q.brute_force_oracle(objective_for(q, spec, "fast"), n)
    assert abs(fit - want_f) <= 1e-9 * abs(want_f)
    exact_of_found = objective_for(q, spec, "exact").evaluate_block(signs[None])[0]
    assert abs(exact_of_found - want_f) <= 1e-9 * abs(want_f)


@pytest.mark.gpu
def test_device_search_beyond_the_reference_limit(q):
    """n = 22 (4.2M patterns, the reference refuses n > 20): device result equals
    the oracle's exhaustive argmax."""
    n = 22
    s = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(s, q.default_dispersion(), 1.0, n, mode="exact")
    signs, fit = q.brute_force_oracle(obj, n, limit=24)
    from paper_2511_01255_b200 import tables as T

    t = T.build_tables("thg", 1.0, n, tuple(q.default_dispersion().mismatches_at(1404.0)))
    prob = O.Problem("thg", t.e1[None], t.b[None], np.array([t.w]), np.array([t.hconst]), t.normalization)
    vals = O.evaluate_block(prob, lex_patterns(n))
    best = int(np.argmax(vals))
    assert np.array_equal(signs, q.lexicographic_signs(best, n))
    assert fit == vals[best]


@pytest.mark.gpu
def test_trials_reproduce_reference_runs(q):
    """run_trials(C1, hybrid, 3 trials from seed 0) = the reference's C1 runs for
    seeds 0, 1, 2 (exact mode: bit-identical final fitness)."""
    rx = golden("runs.npz")
    spec = spec_of(rx, "c1_s0")
    obj = objective_for(q, spec, "exact")
    stats, recs = q.run_trials(obj, "hybrid", 3, 0, dimension=spec["count"], pop_size=spec["NP"],
                               generations=spec["G"], max_concurrent=2)
    want = [float(rx[f"c1_s{s}__best_fit"]) for s in range(3)]
    assert [r.seed for r in recs] == [0, 1, 2]
    assert [r.final_fitness for r in recs] == want
    assert stats.average == float(np.mean(want))
    assert stats.std == float(np.std(want, ddof=1))
    assert stats.maximum == max(want) and stats.minimum == min(want)
    for r in recs:
        assert 0.0 < r.deff_norm and r.time_s > 0.0


@pytest.mark.gpu
def test_trials_equal_lone_runs_all_algorithms(q):
    obj = q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)), q.default_dispersion(), 1.0, 300)
    kw = dict(dimension=300, pop_size=24, generations=30)
    rep = q.compare_algorithms(obj, 10, 5, **kw)
    for algo in q.ALGORITHMS:
        lone = [q.run(algo, obj, seed=5 + t, **kw).best.fitness for t in (0, 4, 9)]
        _, recs = q.run_trials(obj, algo, 10, 5, **kw)
        assert [recs[t].final_fitness for t in (0, 4, 9)] == lone
        assert rep.stats[algo].average == float(np.mean([r.final_fitness for r in recs]))
    assert rep.ratio("hybrid", "de") == rep.stats["hybrid"].average / rep.stats["de"].average
