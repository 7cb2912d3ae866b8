"""Pin the CPU oracle (oracle/) and the host table precompute to the reference.

Every expected value here was produced by the reference package itself
(tests/golden/make_golden.py); comparisons are bit-exact (np.array_equal / ==).
These run on CPU in a few seconds and are the foundation the GPU parity tests
stand on: the GPU tests compare the CUDA engine with this oracle.
"""

import json

import numpy as np
import pytest

from conftest import golden, spec_of, unpack_signs
from oracle import oracle as O
from paper_2511_01255_b200 import tables as T


def problem_from_spec(spec):
    proc = "thg" if spec["variant"].endswith("thg") else "shg"
    tabs = [T.build_tables(proc, spec["thickness"], spec["count"], dk) for dk in spec["dks"]]
    scale = tabs[0].normalization if spec["normalization"] == "normalized" else 1.0
    return O.Problem(proc, np.stack([t.e1 for t in tabs]),
                     np.stack([t.b for t in tabs]) if proc == "thg" else None,
                     np.array([t.w for t in tabs]), np.array([t.hconst for t in tabs]), scale,
                     spec["variant"].startswith("multi"), spec["g0"], spec["beta"])


def settings_from_spec(spec):
    s = O.RunSettings()
    pr = spec.get("params", {})
    if "de_params" in pr:
        d = pr["de_params"]
        s.f_max, s.f_min, s.cr, s.x_min, s.x_max = d["f_max"], d["f_min"], d["cr"], d["x_min"], d["x_max"]
    if "gwo_params" in pr:
        d = pr["gwo_params"]
        s.gwo_a, s.gwo_a_final, s.leader_count = d["a"], d["a_final"], d["leader_count"]
        s.discreteness_factor, s.divide_by_leader_count = d["discreteness_factor"], d["divide_by_leader_count"]
    if "schedules" in pr:
        for k, v in pr["schedules"].items():
            setattr(s, k, v)
    return s


# ---------------------------------------------------------------------------
# rng
# ---------------------------------------------------------------------------

def test_fold_key_and_fill():
    fx = golden("rng.npz")
    paths = json.loads(str(fx["paths"]))
    keys = [O.fold_key(p[0], *p[1:]) for p in paths]
    assert keys == [int(k) for k in fx["keys"]]
    fills = np.concatenate([O.uniform_fill(int(k), int(s), int(n))
                            for k, s, n in zip(fx["keys"], fx["starts"], fx["lens"])])
    assert np.array_equal(fills, fx["fills"])


def test_randint_sequences():
    fx = golden("rng.npz")
    for (seed, path, bound, name) in ((5, 1, 7, "randints"), (3, 9, 1021, "randints_big")):
        u = O.uniform_fill(O.fold_key(seed, path), 0, 500)
        got = np.minimum((u * bound).astype(np.int64), bound - 1)
        assert np.array_equal(got, fx[name])


def test_random_population_matrix():
    fx = golden("rng.npz")
    assert np.array_equal(O.random_population_matrix(8, 40, seed=3), unpack_signs(fx["rpm_packed"], 40))


# ---------------------------------------------------------------------------
# host tables
# ---------------------------------------------------------------------------

def test_mismatches_bit_exact():
    tb = golden("tables.npz")
    disp = T.default_dispersion(25.0)
    got = np.array([tuple(T.phase_mismatches(disp, float(w))) for w in tb["wl64"]])
    assert np.array_equal(got, tb["dk64"])
    got = np.array([tuple(T.phase_mismatches(disp, float(w))) for w in tb["extra_wl"]])
    assert np.array_equal(got, tb["dk_extra"])
    hot = T.default_dispersion(80.0)
    got = np.array([tuple(T.phase_mismatches(hot, float(w))) for w in tb["extra_wl"]])
    assert np.array_equal(got, tb["dk_extra_80c"])
    assert T.refractive_index(disp, 1.064) == float(tb["n_e_1064"])


@pytest.mark.parametrize("case", range(6))
def test_tables_bit_exact(case):
    tb = golden("tables.npz")
    t, n, dk1, dk2 = tb[f"c{case}_args"]
    th = T.build_tables("thg", t, int(n), (dk1, dk2))
    sh = T.build_tables("shg", t, int(n), (dk1, dk2))
    assert np.array_equal(th.e1, tb[f"c{case}_e1"])
    assert np.array_equal(th.b, tb[f"c{case}_b"])
    assert th.w == complex(tb[f"c{case}_w12"])
    assert th.hconst == complex(tb[f"c{case}_hconst"])
    assert th.normalization == float(tb[f"c{case}_norm"])
    assert sh.w == complex(tb[f"c{case}_w1"])
    assert sh.normalization == float(tb[f"c{case}_norm1"])


def test_dispersion_range_errors():
    disp = T.default_dispersion()
    with pytest.raises(ValueError, match="below"):
        T.refractive_index(disp, 0.3)
    with pytest.raises(ValueError, match="above"):
        T.refractive_index(disp, 6.0)
    with pytest.raises(ValueError, match="no mismatch override"):
        T.MismatchTable({1.0: T.PhaseMismatchPair(0, 0)}).mismatches_at(2.0)


# ---------------------------------------------------------------------------
# fitness
# ---------------------------------------------------------------------------

def fitness_names():
    return json.loads(str(golden("fitness.npz")["names"]))


@pytest.mark.parametrize("name", fitness_names())
def test_oracle_fitness_bit_exact(name):
    fx = golden("fitness.npz")
    spec = spec_of(fx, name)
    signs = unpack_signs(fx[f"{name}__signs"], spec["count"])
    proc = "thg" if spec["variant"].endswith("thg") else "shg"
    P = O.Problem(proc, fx[f"{name}__e1"], fx.get(f"{name}__b"), fx[f"{name}__w"], fx.get(f"{name}__h"),
                  float(fx[f"{name}__scale"]), spec["variant"].startswith("multi"), spec["g0"], spec["beta"])
    assert np.array_equal(O.evaluate_block(P, signs), fx[f"{name}__fit"])
    assert np.array_equal(O.sum_block(P, signs), fx[f"{name}__sum0"])
    # tables from our own host precompute give the same values
    assert np.array_equal(O.evaluate_block(problem_from_spec(spec), signs, threads=1), fx[f"{name}__fit"])


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------

def test_de_operators():
    fx = golden("operators.npz")
    for ci in fx["de_cases"]:
        NP, D, f, cr, seed, g = fx[f"de{ci}_args"]
        NP, D, seed, g = int(NP), int(D), int(seed), int(g)
        genome = fx[f"de{ci}_genome"]
        for i in range(NP):
            key = O.fold_key(seed, g, i)
            trial, picks, m, jr = O.de_trial(key, genome, i, float(f), float(cr))
            assert np.array_equal(trial, fx[f"de{ci}_trial"][i])
            assert list(picks) == list(fx[f"de{ci}_picks"][i])
            assert m == fx[f"de{ci}_m"][i]
            assert jr == fx[f"de{ci}_jrand"][i]


def test_gwo_discrete():
    fx = golden("operators.npz")
    for ci in fx["gwo_cases"]:
        D, k, early, pd, psl, pfl, disc, seed, base = fx[f"gwo{ci}_args"]
        out = O.gwo_discrete(int(fx[f"gwo{ci}_key"]), int(base), fx[f"gwo{ci}_leaders"], pd, psl, pfl, disc,
                             bool(early))
        assert np.array_equal(out, fx[f"gwo{ci}_out"])


def test_gwo_continuous():
    fx = golden("operators.npz")
    for ci in fx["gwoc_cases"]:
        D, a, div, seed = fx[f"gwoc{ci}_args"]
        out = O.gwo_continuous(int(fx[f"gwoc{ci}_key"]), fx[f"gwoc{ci}_x"], fx[f"gwoc{ci}_leaders"], float(a),
                               bool(div))
        assert np.array_equal(out, fx[f"gwoc{ci}_out"])


def test_reduce_best():
    fx = golden("operators.npz")
    for ci in range(int(fx["rb_cases"])):
        v = fx[f"rb{ci}_vals"]
        for k in (1, 3, 4, min(10, v.size)):
            assert O.reduce_best(v, k) == list(fx[f"rb{ci}_k{k}"])


def test_numpy_stats_replica():
    fx = golden("operators.npz")
    for ci in fx["st_cases"]:
        x = fx[f"st{ci}_x"]
        mx, mean, std, s, mn = fx[f"st{ci}_res"]
        m2, s2 = O.mean_std(x)
        assert (m2, s2) == (mean, std)
        assert O.pairwise_sum(x) == s


def test_init_population():
    fx = golden("operators.npz")
    assert np.array_equal(O.init_population(5, 6, -1.0, 1.0, 99), fx["init_genome"])
    assert np.array_equal(O.init_population(7, 33, -0.3, 2.5, -4), fx["init_genome2"])


# ---------------------------------------------------------------------------
# full runs, including the reference's own golden_trace_seed7 regression
# ---------------------------------------------------------------------------

def run_names():
    return json.loads(str(golden("runs.npz")["names"]))


@pytest.mark.parametrize("name", run_names())
def test_oracle_runs_bit_exact(name):
    rx = golden("runs.npz")
    spec = spec_of(rx, name)
    trace, bg, bp, bf = O.run(problem_from_spec(spec), spec["algorithm"], spec["NP"], spec["G"], spec["seed"],
                              settings_from_spec(spec))
    assert np.array_equal(trace, rx[f"{name}__trace"])
    assert np.array_equal(bg, rx[f"{name}__best_genome"])
    assert np.array_equal(bp, rx[f"{name}__best_proj"])
    assert bf == float(rx[f"{name}__best_fit"])


def test_oracle_thread_count_invariance():
    rx = golden("runs.npz")
    spec = spec_of(rx, "hyb_k3")
    P = problem_from_spec(spec)
    a = O.run(P, "hybrid", spec["NP"], spec["G"], spec["seed"], settings_from_spec(spec), threads=1)
    b = O.run(P, "hybrid", spec["NP"], spec["G"], spec["seed"], settings_from_spec(spec), threads=5)
    assert np.array_equal(a[0], b[0])
