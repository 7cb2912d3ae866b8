"""GPU: the reference's own tests of the path, run against the device engine.

Mirrors /root/reference/pkg/tests/test_optimizer.py (TestRunDrivers, :339-401),
test_objectives.py (:26-135) and test_rng.py (:7-56) with the same inputs and
assertions, so a user of the reference can read this file as the reference's
suite passing on the B200 drop-in.  Exact mode where the reference compares
with ==; the default fast mode where it compares with a tolerance.
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def q():
    import torch

    torch.cuda.set_device(0)
    import paper_2511_01255_b200 as pkg

    return pkg


def toy_objective(q, mode="fast"):
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    return q.make_objective(spec, q.MismatchTable({1404.0: q.PhaseMismatchPair(0.3, 0.7)}), 1.0, 16, mode=mode)


def random_signs(rng, n):
    return np.where(rng.random(n) < 0.5, -1, 1).astype(np.int8)


# ------------------------------------------------------------ test_optimizer.py TestRunDrivers
class TestRunDrivers:
    def test_zero_generations_returns_initial_best(self, q):
        obj = toy_objective(q, "exact")
        result = q.run_hybrid(obj, dimension=16, pop_size=8, generations=0, seed=3)
        assert len(result.trace) == 1
        from paper_2511_01255_b200 import rng

        # init_population (optimizer.py:207-226): gene j of row i = lo + u_j (hi - lo), stream (seed, 0, i)
        genome = np.stack([-1.0 + rng.uniform_fill(rng.fold_key(3, 0, i), 0, 16) * 2.0 for i in range(8)])
        fits = obj.evaluate_block(np.where(genome >= 0.0, 1, -1).astype(np.int8))
        assert result.best.fitness == pytest.approx(max(fits), rel=1e-15)

    def test_elitism_and_f_bounds(self, q):
        result = q.run_hybrid(toy_objective(q), dimension=16, pop_size=10, generations=25, seed=11)
        best = result.trace_column("best")
        assert np.all(np.diff(best) >= 0)
        f = result.trace_column("f")
        assert np.all((f >= 0.01) & (f <= 0.1 + 1e-15))

    def test_branches_disabled_f_monotone_with_exact_endpoints(self, q):
        sch = q.Schedules(adaptive_branches=False)
        result = q.run_hybrid(toy_objective(q), dimension=16, pop_size=8, generations=20, seed=5, schedules=sch)
        f = result.trace_column("f")
        assert f[0] == pytest.approx(0.1, abs=1e-12)
        assert f[-1] == pytest.approx(0.01, abs=1e-12)
        assert np.all(np.diff(f) <= 1e-15)

    def test_worker_count_does_not_change_trace(self, q):
        obj = toy_objective(q)
        r1 = q.run_hybrid(obj, dimension=16, pop_size=10, generations=15, seed=21, workers=1)
        r4 = q.run_hybrid(obj, dimension=16, pop_size=10, generations=15, seed=21, workers=4)
        assert r1.trace == r4.trace
        assert np.array_equal(r1.best.projection, r4.best.projection)

    def test_seed_changes_trajectory(self, q):
        obj = toy_objective(q)
        r1 = q.run_hybrid(obj, dimension=16, pop_size=10, generations=10, seed=1)
        r2 = q.run_hybrid(obj, dimension=16, pop_size=10, generations=10, seed=2)
        assert r1.trace != r2.trace

    def test_projections_stay_binary_and_size_constant(self, q):
        result = q.run_hybrid(toy_objective(q), dimension=16, pop_size=8, generations=10, seed=9)
        assert set(np.unique(result.best.projection)).issubset({-1, 1})
        assert result.best.projection.size == 16 and result.best.genome.size == 16

    def test_run_de_and_run_gwo_smoke(self, q):
        obj = toy_objective(q)
        rde = q.run_de(obj, dimension=16, pop_size=8, generations=10, seed=13)
        assert len(rde.trace) == 11
        assert np.all(np.diff(rde.trace_column("best")) >= 0)
        rgwo = q.run_gwo(obj, dimension=16, pop_size=8, generations=10, seed=13)
        assert len(rgwo.trace) == 11
        assert rgwo.best.fitness >= rgwo.trace[0][1] - 1e-15

    def test_dispatch_by_name(self, q):
        obj = toy_objective(q)
        for name in ("hybrid", "de", "gwo"):
            result = q.run(name, obj, dimension=16, pop_size=8, generations=5, seed=1)
            assert result.best.fitness is not None
        with pytest.raises(ValueError, match="algorithm"):
            q.run("annealing", obj, dimension=16, pop_size=8, generations=5, seed=1)

    def test_best_individual_is_consistent(self, q):
        """The returned best's fitness is the objective of its projection (exact mode: ==)."""
        obj = toy_objective(q, "exact")
        for name in ("hybrid", "de", "gwo"):
            res = q.run(name, obj, dimension=16, pop_size=12, generations=20, seed=4)
            assert obj(res.best.projection) == res.best.fitness
            assert np.array_equal(res.best.projection, np.where(res.best.genome >= 0.0, 1, -1))


# ------------------------------------------------------------ test_objectives.py
DISPERSIONLESS_COEFFS = {"a1": 4.0}


class TestObjectives:
    def dispersionless(self, q):
        return q.DispersionModel(DISPERSIONLESS_COEFFS, 25.0, (0.2, 5.0))

    def test_spec_validation(self, q):
        with pytest.raises(ValueError, match="variant"):
            q.ObjectiveSpec("shg", (1404.0,))
        with pytest.raises(ValueError):
            q.ObjectiveSpec("single_thg", (1404.0, 1500.0))
        with pytest.raises(ValueError):
            q.ObjectiveSpec("multi_thg", (1404.0,))

    @pytest.mark.parametrize("variant", ["single_shg", "single_thg"])
    def test_all_up_dispersionless_normalized(self, q, variant):
        spec = q.ObjectiveSpec(variant, (1404.0,))
        pattern = q.DomainPattern(1.0, np.ones(50, dtype=np.int8))
        assert q.fitness_single(pattern, spec, self.dispersionless(q)) == pytest.approx(1.0, abs=1e-12)

    def test_variant_mismatch_rejected(self, q):
        spec = q.ObjectiveSpec("multi_shg", (1300.0, 1500.0))
        with pytest.raises(ValueError, match="single"):
            q.fitness_single(q.DomainPattern(1.0, np.ones(4, dtype=np.int8)), spec, self.dispersionless(q))
        spec = q.ObjectiveSpec("single_shg", (1404.0,))
        with pytest.raises(ValueError, match="multi"):
            q.fitness_multi(q.DomainPattern(1.0, np.ones(4, dtype=np.int8)), spec, self.dispersionless(q))

    def test_multi_orientation_negated(self, q):
        spec = q.ObjectiveSpec("multi_shg", (1300.0, 1500.0), g0=10.0, beta=1.0)
        provider = q.MismatchTable({1300.0: q.PhaseMismatchPair(0.0, 0.0), 1500.0: q.PhaseMismatchPair(0.0, 0.0)})
        fit = q.fitness_multi(q.DomainPattern(1.0, np.ones(20, dtype=np.int8)), spec, provider)
        assert fit == pytest.approx(-(2 * 9.0), rel=1e-12)

    def test_block_matches_scalar_calls(self, q):
        rng = np.random.default_rng(31)
        spec = q.ObjectiveSpec("multi_thg", (1300.0, 1500.0), g0=2.0, beta=1.5)
        provider = q.MismatchTable({1300.0: q.PhaseMismatchPair(0.4, 1.1), 1500.0: q.PhaseMismatchPair(-0.2, 0.9)})
        for mode in ("exact", "fast"):
            obj = q.make_objective(spec, provider, 0.5, 24, mode=mode)
            block = np.stack([random_signs(rng, 24) for _ in range(10)])
            fits = obj.evaluate_block(block)
            for row, fit in zip(block, fits):
                assert obj(row) == fit

    def test_gains_and_normalized_gains(self, q):
        spec = q.ObjectiveSpec("single_shg", (1404.0,), normalization="raw")
        obj = q.make_objective(spec, self.dispersionless(q), 1.0, 30)
        signs = np.ones(30, dtype=np.int8)
        assert obj.gains(signs)[0] == pytest.approx(30.0, rel=1e-12)
        assert obj.normalized_gains(signs)[0] == pytest.approx(1.0, rel=1e-12)

    def test_multi_objective_formula(self, q):
        assert q.multi_objective([3.0, 3.0], g0=10.0, beta=1.0) == pytest.approx(14.0)
        assert q.multi_objective([2.0, 4.0], g0=10.0, beta=2.0) == pytest.approx(18.0)
        assert q.multi_objective([4.0], g0=10.0, beta=0.0) == pytest.approx(6.0)
        assert q.multi_objective([0.2, 0.35, 0.4], g0=2.0, beta=1.0) < q.multi_objective([0.2, 0.3, 0.4], g0=2.0,
                                                                                         beta=1.0)
        assert q.multi_objective([0.3, 0.3], g0=2.0, beta=1.0) < q.multi_objective([0.2, 0.4], g0=2.0, beta=1.0)

    def test_single_multi_consistency(self, q):
        spec = q.ObjectiveSpec("single_thg", (1404.0,))
        provider = q.MismatchTable({1404.0: q.PhaseMismatchPair(0.3, 0.7)})
        single = q.fitness_single(q.DomainPattern(1.0, np.ones(12, dtype=np.int8)), spec, provider)
        assert abs(-q.multi_objective([single], g0=0.0, beta=0.0)) == pytest.approx(single)


# ------------------------------------------------------------ test_rng.py (device fill)
class TestRng:
    def test_same_path_reproduces_bit_exactly(self, q):
        from paper_2511_01255_b200 import rng

        a = rng.uniform_fill(rng.fold_key(42, 3, 7), 0, 1000)
        b = rng.uniform_fill(rng.fold_key(42, 3, 7), 0, 1000)
        assert np.array_equal(a, b)

    def test_draws_depend_only_on_counter_not_history(self, q):
        from paper_2511_01255_b200 import rng

        key = rng.fold_key(5, 1)
        whole = rng.uniform_fill(key, 0, 100)
        assert np.array_equal(rng.uniform_fill(key, 40, 60), whole[40:])

    def test_uniform_statistics(self, q):
        from paper_2511_01255_b200 import rng

        u = rng.uniform_fill(rng.fold_key(2024), 0, 200_000)
        assert u.min() >= 0.0 and u.max() < 1.0
        assert abs(u.mean() - 0.5) < 5e-3
        assert abs(u.var() - 1.0 / 12.0) < 5e-3

    def test_negative_and_large_seeds_fold(self, q):
        from paper_2511_01255_b200 import rng

        assert rng.fold_key(-1) == rng.fold_key(2**64 - 1)
        assert math.isfinite(rng.uniform_fill(rng.fold_key(2**70), 0, 1)[0])
