"""GPU parity: the CUDA engine (through the C ABI) against the oracle and the
reference's golden vectors.

Bars (north_star): fitness within 1e-9 relative in fast mode and bit-exact in
exact mode; selection / crossover / leader decisions bit-exact given identical
draws (proved through bit-exact traces and best individuals of full runs);
final best matching the reference's on the reference configs.
"""

import json

import numpy as np
import pytest

from conftest import golden, spec_of, unpack_signs
from oracle import oracle as O
from test_oracle_golden import problem_from_spec, settings_from_spec

pytestmark = pytest.mark.gpu

FAST_RTOL = 1e-9  # north_star: fp64 fitness within 1e-9 relative


@pytest.fixture(scope="module")
def q():
    import torch

    torch.cuda.set_device(0)
    import paper_2511_01255_b200 as pkg

    return pkg


def provider_for(q, spec):
    return q.MismatchTable({float(w): q.PhaseMismatchPair(*dk) for w, dk in zip(spec["pumps"], spec["dks"])})


def objective_for(q, spec, mode):
    s = q.ObjectiveSpec(spec["variant"], tuple(spec["pumps"]), g0=spec["g0"], beta=spec["beta"],
                        normalization=spec["normalization"])
    return q.make_objective(s, provider_for(q, spec), spec["thickness"], spec["count"], mode=mode)


# ---------------------------------------------------------------- rng
def test_uniform_fill_bit_exact(q):
    from paper_2511_01255_b200 import rng

    fx = golden("rng.npz")
    got = np.concatenate([rng.uniform_fill(int(k), int(s), int(n))
                          for k, s, n in zip(fx["keys"], fx["starts"], fx["lens"])])
    assert np.array_equal(got, fx["fills"])
    assert np.array_equal(rng.random_population_matrix(8, 40, seed=3), unpack_signs(fx["rpm_packed"], 40))


def test_uniform_fill_large_vs_oracle(q):
    from paper_2511_01255_b200 import rng

    key = rng.fold_key(123, 4, 5)
    n = 3_000_001
    assert np.array_equal(rng.uniform_fill(key, 2**40 + 3, n), O.uniform_fill(key, 2**40 + 3, n))


# ---------------------------------------------------------------- fitness
FIT_NAMES = json.loads(str(golden("fitness.npz")["names"]))


@pytest.mark.parametrize("name", FIT_NAMES)
def test_fitness_exact_bit_exact(q, name):
    fx = golden("fitness.npz")
    spec = spec_of(fx, name)
    obj = objective_for(q, spec, "exact")
    signs = unpack_signs(fx[f"{name}__signs"], spec["count"])
    assert np.array_equal(obj.evaluate_block(signs), fx[f"{name}__fit"])
    assert np.array_equal(obj.kernel_sums(signs), fx[f"{name}__sum0"])
    assert obj(signs[0]) == fx[f"{name}__fit"][0]
    assert np.array_equal(obj.gains(signs[0]), fx[f"{name}__gains0"])
    assert np.array_equal(obj.normalized_gains(signs[0]), fx[f"{name}__ngains0"])


@pytest.mark.parametrize("name", FIT_NAMES)
def test_fitness_fast_within_tolerance(q, name):
    fx = golden("fitness.npz")
    spec = spec_of(fx, name)
    obj = objective_for(q, spec, "fast")
    signs = unpack_signs(fx[f"{name}__signs"], spec["count"])
    got = obj.evaluate_block(signs)
    want = fx[f"{name}__fit"]
    np.testing.assert_allclose(got, want, rtol=FAST_RTOL, atol=0)


@pytest.mark.parametrize("D,rows,variant,nwl", [(10_000, 300, "single_thg", 1), (100_000, 24, "single_thg", 1),
                                                (20_000, 40, "multi_thg", 64), (3000, 64, "multi_thg", 2),
                                                (12_345, 50, "single_shg", 1), (5, 33, "single_thg", 1)])
def test_fitness_fast_full_size_vs_oracle(q, D, rows, variant, nwl):
    pumps = tuple(float(w) for w in np.linspace(1380.0, 1430.0, nwl)) if nwl > 1 else (1404.0,)
    spec = q.ObjectiveSpec(variant, pumps)
    thick = 0.1 if D == 100_000 else 0.5 if nwl == 64 else 1.0
    obj = q.make_objective(spec, q.default_dispersion(), thick, D, mode="fast")
    signs = O.random_population_matrix(rows, D, seed=D + rows)
    tb = obj.tables
    P = O.Problem(spec.process, np.stack([t.e1 for t in tb]),
                  np.stack([t.b for t in tb]) if spec.process == "thg" else None, np.array([t.w for t in tb]),
                  np.array([t.hconst for t in tb]), tb[0].normalization, spec.is_multi, spec.g0, spec.beta)
    want = O.evaluate_block(P, signs)
    got = obj.evaluate_block(signs)
    np.testing.assert_allclose(got, want, rtol=FAST_RTOL, atol=0)
    exact = obj.evaluate_block(signs, mode="exact")
    assert np.array_equal(exact, want)


def test_fitness_pure_function_of_row_bits(q):
    """Identical rows give identical fitness regardless of batch size/position,
    and the global sign flip is an exact symmetry (optimizer ties depend on it)."""
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, 10_000, mode="fast")
    signs = O.random_population_matrix(64, 10_000, seed=5)
    a = obj.evaluate_block(signs)
    b = obj.evaluate_block(np.concatenate([signs[7:9], signs, signs[::-1]]))
    assert np.array_equal(a, b[2:66])
    assert np.array_equal(a[::-1], b[66:])
    assert np.array_equal(b[0:2], a[7:9])
    assert np.array_equal(obj.evaluate_block(-signs), a)


@pytest.mark.parametrize("D", [300, 2000, 20_000, 70_000])
def test_fitness_fused_finish_batch_invariant(q, D):
    """Single-wavelength fitness is finished by the last segment CTA of each
    128-row block (one stitch run per lane for S <= 32 segments, several for
    S > 32): values are identical whatever the batch size and row position,
    and within 1e-9 of exact mode."""
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, D, mode="fast")
    ex = q.make_objective(spec, q.default_dispersion(), 1.0, D, mode="exact")
    signs = O.random_population_matrix(131, D, seed=D)
    a = obj.evaluate_block(signs)
    for lo, hi in ((0, 1), (5, 133), (130, 131), (3, 131)):
        assert np.array_equal(obj.evaluate_block(signs[lo:hi]), a[lo:hi])
    np.testing.assert_allclose(a, ex.evaluate_block(signs), rtol=FAST_RTOL, atol=0)


def test_evaluate_block_concurrent_threads(q):
    """The reference's parexec calls evaluate_block from worker threads at once
    (parexec.py:88-105): concurrent calls on one objective give the serial values."""
    from concurrent.futures import ThreadPoolExecutor

    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, 4000, mode="fast")
    signs = O.random_population_matrix(256, 4000, seed=11)
    want = obj.evaluate_block(signs)
    chunks = [signs[k:k + 16] for k in range(0, 256, 16)]
    with ThreadPoolExecutor(8) as ex:
        for _ in range(3):
            got = np.concatenate(list(ex.map(obj.evaluate_block, chunks)))
            assert np.array_equal(got, want)


def test_fitness_edge_shapes(q):
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    prov = q.MismatchTable({1404.0: q.PhaseMismatchPair(0.3, 0.7)})
    for D in (1, 2, 3, 4, 127, 128, 129, 255, 256, 257):
        obj = q.make_objective(spec, prov, 1.0, D, mode="fast")
        ex = q.make_objective(spec, prov, 1.0, D, mode="exact")
        signs = O.random_population_matrix(17, D, seed=D)
        np.testing.assert_allclose(obj.evaluate_block(signs), ex.evaluate_block(signs), rtol=FAST_RTOL, atol=1e-300)
    with pytest.raises(ValueError):
        obj.evaluate_block(np.ones((3, 5), dtype=np.int8))
    assert obj.evaluate_block(np.ones((0, 257), dtype=np.int8)).shape == (0,)


# ---------------------------------------------------------------- leaders
def test_reduce_best_bit_exact(q):
    fx = golden("operators.npz")
    for ci in range(int(fx["rb_cases"])):
        v = fx[f"rb{ci}_vals"]
        for k in (1, 3, 4, min(10, v.size)):
            assert q.reduce_best(v, k) == list(fx[f"rb{ci}_k{k}"])
    with pytest.raises(ValueError, match="empty"):
        q.reduce_best([], 1)
    with pytest.raises(ValueError, match="k must be"):
        q.reduce_best([1.0], 2)


# ---------------------------------------------------------------- full runs
RUN_NAMES = json.loads(str(golden("runs.npz")["names"]))


def run_kwargs(q, spec):
    pr = spec.get("params", {})
    kw = {}
    if "de_params" in pr:
        kw["de_params"] = q.DEParams(**pr["de_params"])
    if "gwo_params" in pr:
        kw["gwo_params"] = q.GWOParams(**pr["gwo_params"])
    if "schedules" in pr:
        kw["schedules"] = q.Schedules(**pr["schedules"])
    return kw


@pytest.mark.parametrize("name", RUN_NAMES)
def test_run_exact_bit_exact(q, name):
    """Exact mode reproduces the reference's traces and best individuals bit-for-bit
    (golden7 is the reference's own golden_trace_seed7 regression)."""
    rx = golden("runs.npz")
    spec = spec_of(rx, name)
    obj = objective_for(q, spec, "exact")
    res = q.run(spec["algorithm"], obj, dimension=spec["count"], pop_size=spec["NP"], generations=spec["G"],
                seed=spec["seed"], **run_kwargs(q, spec))
    trace = np.array(res.trace, dtype=np.float64)
    assert np.array_equal(trace, rx[f"{name}__trace"])
    assert np.array_equal(res.best.genome, rx[f"{name}__best_genome"])
    assert np.array_equal(res.best.projection, rx[f"{name}__best_proj"])
    assert res.best.fitness == float(rx[f"{name}__best_fit"])


@pytest.mark.parametrize("name", ["golden7", "c1_s0", "c1_s1", "c1_s2", "de_small", "gwo_small", "hyb_multi2"])
def test_run_fast_matches_reference(q, name):
    """Fast fitness keeps the reference's trajectory: same best pattern, best
    fitness within 1e-9 relative."""
    rx = golden("runs.npz")
    spec = spec_of(rx, name)
    obj = objective_for(q, spec, "fast")
    res = q.run(spec["algorithm"], obj, dimension=spec["count"], pop_size=spec["NP"], generations=spec["G"],
                seed=spec["seed"], **run_kwargs(q, spec))
    want = float(rx[f"{name}__best_fit"])
    assert abs(res.best.fitness - want) <= FAST_RTOL * abs(want)
    assert np.array_equal(res.best.projection, rx[f"{name}__best_proj"])
    np.testing.assert_allclose(np.array(res.trace), rx[f"{name}__trace"], rtol=FAST_RTOL, atol=1e-15)


def test_graph_and_eager_identical(q):
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, 700, mode="fast")
    de, gwo, sch = q.DEParams(), q.GWOParams(), q.Schedules()
    out = []
    for use_graph in (True, False):
        eng = q.Engine(obj, "hybrid", pop_size=37, generations=30, seed=3, de=de, gwo=gwo, sch=sch)
        eng.init()
        if use_graph:
            eng.prepare(13)
        eng.step(13, use_graph=use_graph)
        eng.step(17, use_graph=use_graph)
        eng.finalize()
        out.append((eng.trace(), eng.population()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1][0], out[1][1][0])


def test_c2_shape_generation_vs_oracle(q):
    """Full-size C2 shape (NP 1024, D 10^4): exact-mode generations equal the oracle's."""
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, 10_000, mode="exact")
    G, stop = 1000, 3
    eng = q.Engine(obj, "hybrid", pop_size=1024, generations=G, seed=0, de=q.DEParams(), gwo=q.GWOParams(),
                   sch=q.Schedules())
    eng.init()
    eng.step(stop)
    t = obj.tables[0]
    P = O.Problem("thg", t.e1[None], t.b[None], np.array([t.w]), np.array([t.hconst]), t.normalization)
    trace, *_ = O.run(P, "hybrid", 1024, G, 0, stop_after=stop)
    assert np.array_equal(eng.trace(0, stop + 1), trace)


def test_validation_errors(q):
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.MismatchTable({1404.0: q.PhaseMismatchPair(0.3, 0.7)}), 1.0, 16)
    with pytest.raises(ValueError, match=">= 4"):
        q.run_hybrid(obj, dimension=16, pop_size=3, generations=2, seed=0)
    with pytest.raises(ValueError, match="algorithm"):
        q.run("annealing", obj, dimension=16, pop_size=8, generations=2, seed=0)
    with pytest.raises(ValueError, match="leader_count"):
        q.GWOParams(leader_count=5)
    with pytest.raises(ValueError, match="cr"):
        q.DEParams(cr=1.5)
    r = q.run_hybrid(obj, dimension=16, pop_size=8, generations=0, seed=3)
    assert len(r.trace) == 1


@pytest.mark.parametrize("algorithm", ["hybrid", "de", "gwo"])
@pytest.mark.parametrize("D,NP", [(2050, 5), (4097, 13), (6000, 7), (40_000, 6)])
def test_odd_shapes_exact_vs_oracle(q, algorithm, D, NP):
    """Row lengths around the trial's chunk / stage / word boundaries (2,050:
    stages of 1,024 + 1,024 + 128 genes; 4,097: a 1-gene tail past a chunk;
    6,000: a partial second chunk; 40,000: the 8,192-gene chunks of long rows)
    and tiny odd populations: exact-mode runs
    equal the oracle bit for bit (trace, best genome, projection, fitness)."""
    G, seed = 12, 5
    spec = q.ObjectiveSpec("single_thg", (1404.0,))
    obj = q.make_objective(spec, q.default_dispersion(), 1.0, D, mode="exact")
    res = q.run(algorithm, obj, dimension=D, pop_size=NP, generations=G, seed=seed)
    t = obj.tables[0]
    P = O.Problem("thg", t.e1[None], t.b[None], np.array([t.w]), np.array([t.hconst]), t.normalization)
    trace, bg, bp, bf = O.run(P, algorithm, NP, G, seed)
    assert np.array_equal(np.array(res.trace, dtype=np.float64), trace)
    assert np.array_equal(res.best.genome, bg)
    assert np.array_equal(res.best.projection, bp)
    assert res.best.fitness == bf
