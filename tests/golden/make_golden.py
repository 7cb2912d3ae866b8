"""Generate the golden fixtures by running the reference package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports `qpmdesign` from /root/reference/pkg/src (numba backend), evaluates
the hot-path functions on seeded inputs and writes small .npz fixtures next to
this script.  The fixtures are what pins both the CPU oracle (oracle/) and the
CUDA engine; nothing at test time reads /root/reference.

Every array is computed by the reference's own public functions; the names of
the functions used are recorded in each fixture's `meta` string.
"""

import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

import qpmdesign  # noqa: E402
from qpmdesign import _kernels, bench, optimizer, parexec, physics, rng  # noqa: E402
from qpmdesign.objectives import ObjectiveSpec, make_objective  # noqa: E402
from qpmdesign.physics import (  # noqa: E402
    MismatchTable, PhaseMismatchPair, ShgEvaluator, ThgEvaluator, default_dispersion,
)

assert _kernels.backend() == "numba", "golden vectors are recorded for the numba backend"


def packbits(signs2d):
    """int8 +/-1 rows -> little-endian bit rows (bit = 1 for -1)."""
    bits = (np.asarray(signs2d) < 0).astype(np.uint8)
    return np.packbits(bits, axis=-1, bitorder="little")


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


# ---------------------------------------------------------------------------
# rng.py: fold_key, uniform_fill, randint
# ---------------------------------------------------------------------------

def gen_rng():
    paths = [(0,), (7,), (7, 0, 3), (-17, 2), (123, 4, 5), ((1 << 63) + 5, 1, 2), (-1,), (99, 0, 2),
             (11, 4, 6), (2**64 - 1, 2**40, 3)]
    keys = np.array([rng.fold_key(p[0], *p[1:]) for p in paths], dtype=np.uint64)
    path_tbl = np.zeros((len(paths), 3), dtype=object)
    flat_paths = json.dumps([list(p) for p in paths])
    fills = []
    starts = [0, 0, 5, 1000, 2**33, 0, 17, 3, 0, 123456789]
    lens = [64, 333, 10, 100, 50, 7, 1, 129, 1000, 20]
    for key, st, n in zip(keys, starts, lens):
        fills.append(_kernels.uniform_fill(int(key), st, n))
    s = rng.stream(5, 1)
    randints = np.array([s.randint(7) for _ in range(500)], dtype=np.int64)
    s = rng.stream(3, 9)
    randints_big = np.array([s.randint(1021) for _ in range(500)], dtype=np.int64)
    rpm = bench.random_population_matrix(8, 40, seed=3)
    del path_tbl
    save("rng.npz", keys=keys, paths=np.array(flat_paths), starts=np.array(starts, dtype=np.uint64),
         lens=np.array(lens), fills=np.concatenate(fills), randints=randints, randints_big=randints_big,
         rpm_packed=packbits(rpm), meta=np.array("rng.fold_key, _kernels.uniform_fill, CounterStream.randint, "
                                                 "bench.random_population_matrix(8, 40, seed=3)"))


# ---------------------------------------------------------------------------
# physics.py: mismatches and evaluator tables
# ---------------------------------------------------------------------------

TABLE_CASES = [
    # (thickness, count, dk1, dk2)
    (1.0, 64, 0.3, 0.7),
    (1.0, 1000, None, None),  # C1: 1404 nm Sellmeier
    (0.5, 37, 1e-9, 2e-7),  # series branches of _m0/_phi
    (0.1, 200, 0.41937765532544447, 1.2723419565740617),
    (3.0, 50, 0.0, 0.0),
    (2.0, 17, -0.2, 0.9),
]


def gen_tables():
    disp = default_dispersion(25.0)
    wl = np.linspace(1380.0, 1430.0, 64)
    dks = np.array([tuple(physics.phase_mismatches(disp, float(w))) for w in wl])
    extra_wl = np.array([1210.0, 1404.0, 1550.0, 1283.0, 1364.0, 1568.0, 1650.0, 2080.0, 4500.0])
    dks_extra = np.array([tuple(physics.phase_mismatches(disp, float(w))) for w in extra_wl])
    dks_hot = np.array([tuple(physics.phase_mismatches(default_dispersion(80.0), float(w))) for w in extra_wl])
    n_e = physics.refractive_index(disp, 1.064)
    out = dict(wl64=wl, dk64=dks, extra_wl=extra_wl, dk_extra=dks_extra, dk_extra_80c=dks_hot,
               n_e_1064=np.array(n_e))
    for c, (t, n, dk1, dk2) in enumerate(TABLE_CASES):
        if dk1 is None:
            dk1, dk2 = physics.phase_mismatches(disp, 1404.0)
        ev = ThgEvaluator(t, n, PhaseMismatchPair(dk1, dk2))
        sv = ShgEvaluator(t, n, dk1)
        out[f"c{c}_args"] = np.array([t, n, dk1, dk2])
        out[f"c{c}_e1"] = ev._e1
        out[f"c{c}_b"] = ev._b
        out[f"c{c}_w12"] = np.array(ev._w12)
        out[f"c{c}_hconst"] = np.array(ev._hconst)
        out[f"c{c}_norm"] = np.array(ev.normalization)
        out[f"c{c}_w1"] = np.array(sv._w1)
        out[f"c{c}_norm1"] = np.array(sv.normalization)
        assert np.array_equal(sv._e1, ev._e1)
    out["meta"] = np.array("physics.phase_mismatches, refractive_index, ThgEvaluator/ShgEvaluator tables")
    save("tables.npz", **out)


# ---------------------------------------------------------------------------
# objectives.py: evaluate_block on bench.random_population_matrix rows
# ---------------------------------------------------------------------------

def objective_cases():
    disp = default_dispersion(25.0)
    cases = []
    # name, spec, provider, thickness, count, rows
    mt = MismatchTable({1404.0: PhaseMismatchPair(0.3, 0.7)})
    cases.append(("thg_toy", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 64, 40))
    cases.append(("thg_c1", ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, 1000, 48))
    cases.append(("thg_raw", ObjectiveSpec("single_thg", (1404.0,), normalization="raw"), mt, 1.0, 65, 20))
    for n in (1, 2, 7, 8, 31, 32, 33, 63, 127, 129, 300):
        cases.append((f"thg_n{n}", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, n, 9))
    cases.append(("shg_c1", ObjectiveSpec("single_shg", (1404.0,)), disp, 1.0, 1000, 24))
    cases.append(("shg_raw", ObjectiveSpec("single_shg", (1404.0,), normalization="raw"), mt, 1.0, 77, 12))
    cases.append(("multi_thg2", ObjectiveSpec("multi_thg", (1404.0, 1650.0)), disp, 3.0, 300, 16))
    cases.append(("multi_shg5", ObjectiveSpec("multi_shg", (1283.0, 1364.0, 1404.0, 1568.0, 1650.0)), disp, 3.0,
                  300, 16))
    wl64 = tuple(float(w) for w in np.linspace(1380.0, 1430.0, 64))
    cases.append(("multi_thg64", ObjectiveSpec("multi_thg", wl64), disp, 0.5, 400, 12))
    cases.append(("multi_thg9_raw", ObjectiveSpec("multi_thg", wl64[:9], g0=3.0, beta=0.5, normalization="raw"),
                  disp, 0.5, 60, 10))
    return cases


def spec_record(spec, provider, t, n):
    pairs = [tuple(provider.mismatches_at(w)) for w in spec.pump_wavelengths_nm]
    return dict(variant=spec.variant, pumps=list(spec.pump_wavelengths_nm), g0=spec.g0, beta=spec.beta,
                normalization=spec.normalization, thickness=t, count=n, dks=pairs)


def gen_fitness():
    out = {}
    names = []
    for ci, (name, spec, provider, t, n, rows) in enumerate(objective_cases()):
        obj = make_objective(spec, provider, t, n)
        signs = bench.random_population_matrix(rows, n, seed=100 + ci)
        vals = obj.evaluate_block(signs)
        single = np.array([obj(signs[r]) for r in range(rows)])
        assert np.array_equal(single, vals)
        rec = spec_record(spec, provider, t, n)
        out[f"{name}__spec"] = np.array(json.dumps(rec))
        out[f"{name}__signs"] = packbits(signs)
        out[f"{name}__fit"] = vals
        # raw kernel complex sums and per-wavelength tables for wavelength 0
        ev = obj._evaluators[0]
        out[f"{name}__e1"] = np.stack([e._e1 for e in obj._evaluators])
        if spec.process == "thg":
            out[f"{name}__b"] = np.stack([e._b for e in obj._evaluators])
            out[f"{name}__w"] = np.array([e._w12 for e in obj._evaluators])
            out[f"{name}__h"] = np.array([e._hconst for e in obj._evaluators])
            blk = np.empty(rows, dtype=np.complex128)
            _kernels.thg_block(signs, ev._e1, ev._b, blk)
        else:
            out[f"{name}__w"] = np.array([e._w1 for e in obj._evaluators])
            blk = np.empty(rows, dtype=np.complex128)
            _kernels.shg_block(signs, ev._e1, blk)
        out[f"{name}__scale"] = np.array(obj._scale)
        out[f"{name}__sum0"] = blk
        out[f"{name}__gains0"] = obj.gains(signs[0])
        out[f"{name}__ngains0"] = obj.normalized_gains(signs[0])
        names.append(name)
    out["names"] = np.array(json.dumps(names))
    out["meta"] = np.array("objectives.make_objective(...).evaluate_block on bench.random_population_matrix"
                           "(rows, n, seed=100+case); _kernels.thg_block/shg_block")
    save("fitness.npz", **out)


# ---------------------------------------------------------------------------
# optimizer.py operators, parexec.reduce_best, numpy stats
# ---------------------------------------------------------------------------

def gen_operators():
    out = {}
    # --- DE: de_mutate + de_crossover on a seeded population ---
    de_cases = []
    for ci, (NP, D, f, cr, seed, g) in enumerate([(9, 37, 0.1, 0.9, 3, 1), (4, 5, 0.05, 0.5, 1, 7),
                                                  (50, 64, 0.0731, 0.9, 7, 3), (200, 129, 0.01, 0.0, 11, 2),
                                                  (6, 12, 1.7, 1.0, 5, 9)]):
        pop = optimizer.init_population(NP, D, (-1.0, 1.0), seed)
        genome = np.stack([ind.genome for ind in pop.individuals])
        params = optimizer.DEParams(f=min(max(f, 0.01), 2.0), f_min=0.01, f_max=2.0, cr=cr) if f > 0.1 else \
            optimizer.DEParams(f=max(f, 0.01), cr=cr)
        trials, picks, ms, jr = [], [], [], []
        for i in range(NP):
            st = rng.stream(seed, g, i)
            mutant = optimizer.de_mutate(pop, i, params, st)
            m = st._pos
            trial = optimizer.de_crossover(pop.individuals[i].genome, mutant, params.cr, st)
            twin = rng.stream(seed, g, i)
            chosen, pk = {i}, []
            while len(pk) < 3:
                r = twin.randint(NP)
                if r not in chosen:
                    chosen.add(r)
                    pk.append(r)
            jr.append(twin.randint(D))
            trials.append(trial)
            picks.append(pk)
            ms.append(m)
        out[f"de{ci}_args"] = np.array([NP, D, params.f, params.cr, seed, g])
        out[f"de{ci}_genome"] = genome
        out[f"de{ci}_trial"] = np.stack(trials)
        out[f"de{ci}_picks"] = np.array(picks)
        out[f"de{ci}_m"] = np.array(ms)
        out[f"de{ci}_jrand"] = np.array(jr)
        de_cases.append(ci)
    out["de_cases"] = np.array(de_cases)

    # --- GWO discrete ---
    gw = []
    for ci, (D, k, early, pd, psl, pfl, disc, seed) in enumerate([
            (40, 4, True, 0.1, 0.05, 0.02, 1.0, 1), (40, 4, False, 0.1, 0.05, 0.02, 1.0, 2),
            (257, 3, True, 0.3, 0.2, 0.1, 1.0, 3), (257, 3, False, 0.3, 0.2, 0.25, 0.7, 4),
            (1000, 4, False, 0.0, 1.0, 0.0, 1.0, 5), (1000, 4, True, 1.0, 0.0, 0.0, 0.4, 6),
            (64, 4, False, 0.05, 0.025, 0.01, 1.0, 7)]):
        lead_genomes = optimizer.init_population(max(k, 4), D, (-1.0, 1.0), 1000 + ci).individuals[:k]
        if ci == 6:  # exact ties in the late majority vote need an even split
            half = np.where(np.arange(D) % 2 == 0, 1.0, -1.0)
            lead_genomes = [optimizer.Individual.from_genome(v) for v in (half, -half, half, -half)]
        wolf = optimizer.Individual.from_genome(np.zeros(D))
        params = optimizer.GWOParams(leader_count=k, p_dist=pd, p_sl=psl, p_flip=pfl, discreteness_factor=disc)
        st = rng.stream(seed, 2, 5)
        skip = 3 + (ci % 3)
        st.uniforms(skip + 1 + D)  # the DE draws that precede the wolf block
        base = st._pos
        new = optimizer.gwo_discrete_update(wolf, lead_genomes, params, early, st)
        out[f"gwo{ci}_args"] = np.array([D, k, int(early), pd, psl, pfl, disc, seed, base])
        out[f"gwo{ci}_leaders"] = np.stack([l.projection for l in lead_genomes])
        out[f"gwo{ci}_key"] = np.array(rng.fold_key(seed, 2, 5), dtype=np.uint64)
        out[f"gwo{ci}_out"] = new
        gw.append(ci)
    out["gwo_cases"] = np.array(gw)

    # --- GWO continuous (run_gwo) ---
    gc = []
    for ci, (D, a, div, seed) in enumerate([(30, 2.0, False, 1), (30, 0.1, True, 2), (300, 1.3, False, 3),
                                            (5, 0.0, False, 4)]):
        pop = optimizer.init_population(4, D, (-1.0, 1.0), 2000 + ci)
        leaders = pop.individuals[:3]
        wolf = pop.individuals[3]
        if ci == 3:
            leaders = [optimizer.Individual.from_genome(np.zeros(D)) for _ in range(3)]
            wolf = optimizer.Individual.from_genome(np.zeros(D))
        st = rng.stream(seed, 6, 1)
        new = optimizer.gwo_reference_update(wolf, leaders, a, st, div)
        out[f"gwoc{ci}_args"] = np.array([D, a, int(div), seed])
        out[f"gwoc{ci}_x"] = wolf.genome
        out[f"gwoc{ci}_leaders"] = np.stack([l.genome for l in leaders])
        out[f"gwoc{ci}_key"] = np.array(rng.fold_key(seed, 6, 1), dtype=np.uint64)
        out[f"gwoc{ci}_out"] = new
        gc.append(ci)
    out["gwoc_cases"] = np.array(gc)

    # --- reduce_best ---
    r = np.random.default_rng(5)
    vals = [r.integers(0, 50, size=777).astype(float), r.random(10_000), np.full(13, 2.5),
            np.array([5.0, 9.0, 1.0, 7.0, 7.0]), r.standard_normal(8192)]
    for ci, v in enumerate(vals):
        out[f"rb{ci}_vals"] = v
        for k in (1, 3, 4, min(10, v.size)):
            out[f"rb{ci}_k{k}"] = np.array(parexec.reduce_best(v, k, workers=1))
    out["rb_cases"] = np.array(len(vals))

    # --- numpy stats used by the loop (np.max/mean/std) ---
    stats = []
    for ci, n in enumerate([4, 5, 8, 9, 50, 96, 128, 129, 1000, 1020, 1024, 2044, 4096, 8192, 8193]):
        x = r.standard_normal(n) * 0.01 + 0.2
        out[f"st{ci}_x"] = x
        out[f"st{ci}_res"] = np.array([np.max(x), np.mean(x), np.std(x), np.sum(x), np.min(x)])
        stats.append(ci)
    out["st_cases"] = np.array(stats)

    # --- adaptive_f_update ---
    af = []
    for ci, (g, tot, pstd, rng_, conv, base, adapt) in enumerate([
            (0, 100, 0.2, 10.0, 1.0, 1.0, True), (100, 100, 0.2, 10.0, 1.0, 1.0, True),
            (50, 100, 0.01, 10.0, 1.0, 1.0, True), (50, 100, 0.3, 0.5, 1.0, 1.0, True),
            (17, 500, 0.001, 0.002, 0.05, 0.013, True), (250, 500, 0.9, 0.001, 0.5, 0.013, True),
            (7, 9, 0.0, 0.0, 0.0, 0.0, False), (333, 1000, 0.02, 0.03, 0.1, 0.01, True)]):
        sch = optimizer.Schedules(adaptive_branches=adapt)
        st = optimizer.AdaptiveState(generation=g, total_generations=tot, pop_std=pstd, fit_range=rng_,
                                     convergence_rate=conv, decay_coeff=sch.decay_coeff(g, tot),
                                     baseline_std=base)
        f = optimizer.adaptive_f_update(st, optimizer.DEParams(), sch)
        out[f"af{ci}_args"] = np.array([g, tot, pstd, rng_, conv, base, float(adapt), st.decay_coeff])
        out[f"af{ci}_f"] = np.array(f)
        af.append(ci)
    out["af_cases"] = np.array(af)

    # --- init_population ---
    pop = optimizer.init_population(5, 6, (-1.0, 1.0), seed=99)
    out["init_genome"] = np.stack([ind.genome for ind in pop.individuals])
    pop = optimizer.init_population(7, 33, (-0.3, 2.5), seed=-4)
    out["init_genome2"] = np.stack([ind.genome for ind in pop.individuals])
    out["meta"] = np.array("optimizer.de_mutate/de_crossover/gwo_discrete_update/gwo_reference_update/"
                           "init_population/adaptive_f_update, parexec.reduce_best, numpy stats")
    save("operators.npz", **out)


# ---------------------------------------------------------------------------
# full runs (run_hybrid / run_de / run_gwo)
# ---------------------------------------------------------------------------

def run_cases():
    disp = default_dispersion(25.0)
    mt = MismatchTable({1404.0: PhaseMismatchPair(0.3, 0.7)})
    wl64 = tuple(float(w) for w in np.linspace(1380.0, 1430.0, 64))
    C = []
    # name, algorithm, spec, provider, t, n, NP, G, seed, kwargs
    C.append(("golden7", "hybrid", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 64, 50, 50, 7, {}))
    for seed in (0, 1, 2):
        C.append((f"c1_s{seed}", "hybrid", ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, 1000, 50, 500,
                  seed, {}))
    C.append(("de_small", "de", ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, 300, 24, 60, 3, {}))
    C.append(("gwo_small", "gwo", ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, 300, 24, 40, 4, {}))
    C.append(("gwo_desk", "gwo", ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, 200, 20, 40, 5,
              dict(gwo_params=optimizer.GWOParams(a=0.1, a_final=0.01, divide_by_leader_count=True))))
    C.append(("hyb_k3", "hybrid", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 100, 16, 40, 9,
              dict(gwo_params=optimizer.GWOParams(leader_count=3, discreteness_factor=0.8),
                   schedules=optimizer.Schedules(adaptive_branches=False, conv_window=3))))
    C.append(("hyb_shg", "hybrid", ObjectiveSpec("single_shg", (1404.0,)), disp, 1.0, 150, 12, 30, 10,
              dict(de_params=optimizer.DEParams(f=0.05, cr=0.7, f_max=0.05, f_min=0.02))))
    C.append(("hyb_multi2", "hybrid", ObjectiveSpec("multi_thg", (1404.0, 1650.0)), disp, 3.0, 120, 12, 25, 11,
              {}))
    C.append(("hyb_multi64", "hybrid", ObjectiveSpec("multi_thg", wl64), disp, 0.5, 80, 8, 10, 12, {}))
    C.append(("hyb_oracle12", "hybrid", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 12, 64, 200, 0, {}))
    C.append(("hyb_np4", "hybrid", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 1, 4, 12, 2, {}))
    C.append(("hyb_g0", "hybrid", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 16, 8, 0, 3, {}))
    # extreme operator settings (the reference's unit tests probe these branches)
    thg = ObjectiveSpec("single_thg", (1404.0,))
    S = optimizer.Schedules
    C.append(("hyb_cr1", "hybrid", thg, disp, 1.0, 200, 16, 30, 21, dict(de_params=optimizer.DEParams(cr=1.0))))
    C.append(("hyb_cr0", "hybrid", thg, disp, 1.0, 200, 16, 30, 22, dict(de_params=optimizer.DEParams(cr=0.0))))
    C.append(("hyb_dist1", "hybrid", thg, disp, 1.0, 200, 16, 30, 23, dict(schedules=S(p_dist0=1.0, p_sl0=0.0))))
    C.append(("hyb_sl1", "hybrid", thg, disp, 1.0, 200, 16, 30, 24, dict(schedules=S(p_sl0=1.0))))
    C.append(("hyb_flip1", "hybrid", thg, disp, 1.0, 200, 16, 30, 25,
              dict(schedules=S(p_flip0=1.0, phase_split=0.2))))
    C.append(("hyb_all_late", "hybrid", thg, disp, 1.0, 200, 16, 30, 26, dict(schedules=S(phase_split=0.0))))
    C.append(("hyb_all_early", "hybrid", thg, disp, 1.0, 200, 16, 30, 27, dict(schedules=S(phase_split=1.0))))
    C.append(("hyb_fconst", "hybrid", thg, disp, 1.0, 200, 16, 30, 28,
              dict(de_params=optimizer.DEParams(f=0.05, f_min=0.05, f_max=0.05))))
    C.append(("hyb_zero_bounds", "hybrid", thg, disp, 1.0, 64, 8, 10, 29,
              dict(de_params=optimizer.DEParams(x_min=0.0, x_max=0.0))))
    C.append(("hyb_k3_d1", "hybrid", thg, disp, 1.0, 200, 16, 30, 30,
              dict(gwo_params=optimizer.GWOParams(leader_count=3))))
    C.append(("hyb_k4_d06", "hybrid", thg, disp, 1.0, 200, 16, 30, 31,
              dict(gwo_params=optimizer.GWOParams(discreteness_factor=0.6))))
    return C


def gen_runs():
    out = {}
    names = []
    for name, algo, spec, provider, t, n, NP, G, seed, kw in run_cases():
        obj = make_objective(spec, provider, t, n)
        t0 = time.perf_counter()
        res = optimizer.run(algo, obj, dimension=n, pop_size=NP, generations=G, seed=seed, **kw)
        dt = time.perf_counter() - t0
        rec = spec_record(spec, provider, t, n)
        rec.update(algorithm=algo, NP=NP, G=G, seed=seed, seconds=dt)
        params = {}
        for key, v in kw.items():
            params[key] = {f: getattr(v, f) for f in v.__dataclass_fields__}
        rec["params"] = params
        out[f"{name}__spec"] = np.array(json.dumps(rec))
        out[f"{name}__trace"] = np.array(res.trace, dtype=np.float64)
        out[f"{name}__best_genome"] = res.best.genome
        out[f"{name}__best_proj"] = res.best.projection
        out[f"{name}__best_fit"] = np.array(res.best.fitness)
        names.append(name)
        print(f"  {name}: {dt:.2f}s best={res.best.fitness!r}")
    # the reference's own regression file must agree with what we recorded
    golden = np.loadtxt("/root/reference/pkg/tests/data/golden_trace_seed7.csv", delimiter=",", skiprows=1,
                        usecols=1)
    assert np.array_equal(out["golden7__trace"][:, 1], golden)
    out["names"] = np.array(json.dumps(names))
    out["meta"] = np.array("optimizer.run(algorithm, make_objective(...), ...) traces and best individuals; "
                           "golden7 equals pkg/tests/data/golden_trace_seed7.csv")
    save("runs.npz", **out)


# ---------------------------------------------------------------------------
# bench.py: brute_force_oracle (exhaustive optimum, lexicographic tie-break)
# ---------------------------------------------------------------------------

def search_cases():
    disp = default_dispersion(25.0)
    mt = MismatchTable({1404.0: PhaseMismatchPair(0.3, 0.7)})
    return [
        ("thg_toy10", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 10),
        ("thg_c1_12", ObjectiveSpec("single_thg", (1404.0,)), disp, 1.0, 12),
        ("shg_9", ObjectiveSpec("single_shg", (1404.0,)), disp, 2.0, 9),
        ("multi_thg2_11", ObjectiveSpec("multi_thg", (1404.0, 1650.0)), disp, 3.0, 11),
        ("thg_raw_7", ObjectiveSpec("single_thg", (1404.0,), normalization="raw"), mt, 1.0, 7),
        ("thg_1", ObjectiveSpec("single_thg", (1404.0,)), mt, 1.0, 1),
    ]


def gen_search():
    out = {}
    names = []
    for name, spec, provider, t, n in search_cases():
        obj = make_objective(spec, provider, t, n)
        signs, fit = bench.brute_force_oracle(obj, n)
        index = int(sum(int(s < 0) << (n - 1 - j) for j, s in enumerate(signs)))
        assert np.array_equal(bench.lexicographic_signs(index, n), signs)
        out[f"{name}__spec"] = np.array(json.dumps(spec_record(spec, provider, t, n)))
        out[f"{name}__index"] = np.array(index)
        out[f"{name}__fit"] = np.array(fit)
        names.append(name)
        print(f"  {name}: index={index} fit={fit!r}")
    out["names"] = np.array(json.dumps(names))
    out["meta"] = np.array("bench.brute_force_oracle(make_objective(...), n): optimum index and fitness")
    save("search.npz", **out)


# ---------------------------------------------------------------------------
# physics.py: sweep_spectrum over pump wavelengths
# ---------------------------------------------------------------------------

def gen_spectra():
    disp = default_dispersion(25.0)
    out = {}
    names = []
    cases = [("thg_d1000", "thg", 1.0, 1000, 11, np.linspace(1250.0, 1700.0, 19)),
             ("shg_d1000", "shg", 1.0, 1000, 12, np.linspace(1250.0, 1700.0, 19)),
             ("thg_d4096_t05", "thg", 0.5, 4096, 13, np.linspace(1380.0, 1430.0, 64)),
             ("shg_d33", "shg", 2.0, 33, 14, np.array([1404.0, 1300.0, 1550.0]))]
    for name, process, t, n, seed, wls in cases:
        signs = bench.random_population_matrix(1, n, seed)[0]
        pattern = physics.DomainPattern(t, signs)
        rows = physics.sweep_spectrum(pattern, disp, list(wls), process)
        out[f"{name}__spec"] = np.array(json.dumps(dict(process=process, thickness=t, count=n, seed=seed)))
        out[f"{name}__signs"] = np.asarray(signs, dtype=np.int8)
        out[f"{name}__rows"] = np.array(rows, dtype=np.float64)
        names.append(name)
        print(f"  {name}: {len(rows)} wavelengths, max |d| {max(r[1] for r in rows):.6g}")
    out["names"] = np.array(json.dumps(names))
    out["meta"] = np.array("physics.sweep_spectrum(DomainPattern(t, bench.random_population_matrix(1, n, seed)[0]), "
                           "default_dispersion(25.0), wavelengths, process) rows (wl, |d|, |d|/norm)")
    save("spectra.npz", **out)


if __name__ == "__main__":
    print("qpmdesign", qpmdesign.__version__, "backend", _kernels.backend(), "numpy", np.__version__)
    only = sys.argv[1:]
    for name, fn in (("rng", gen_rng), ("tables", gen_tables), ("fitness", gen_fitness),
                     ("operators", gen_operators), ("runs", gen_runs), ("search", gen_search),
                     ("spectra", gen_spectra)):
        if not only or name in only:
            fn()
