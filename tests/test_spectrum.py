"""batched spectra (physics.sweep_spectrum).

CPU: the host tables (tables.py) and the oracle's kernel sums reproduce the
reference's sweep_spectrum rows bit-exactly (tests/golden/spectra.npz).
GPU: the device sweep (phase tables generated in the kernel) agrees with the
reference rows to 1e-10 relative, for single patterns and batched.
"""

import json

import numpy as np
import pytest

from conftest import golden, spec_of
from oracle import oracle as O
from paper_2511_01255_b200 import tables as T

NAMES = json.loads(str(golden("spectra.npz")["names"]))
RTOL = 1e-10


def reference_rows(name):
    fx = golden("spectra.npz")
    return spec_of(fx, name), fx[f"{name}__signs"], fx[f"{name}__rows"]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_spectrum_matches_reference(name):
    spec, signs, rows = reference_rows(name)
    disp = T.default_dispersion(25.0)
    for wl, mag, norm_mag in rows:
        t = T.build_tables(spec["process"], spec["thickness"], spec["count"], disp.mismatches_at(wl))
        prob = O.Problem(spec["process"], t.e1[None], t.b[None] if t.b is not None else None,
                         np.array([t.w]), np.array([t.hconst]), 1.0)
        acc = O.sum_block(prob, signs[None])[0]
        d = acc * t.w + t.hconst if spec["process"] == "thg" else complex(acc * t.w)
        assert abs(d) == mag
        assert abs(d) / t.normalization == norm_mag


def test_spectrum_validation():
    import paper_2511_01255_b200 as q

    pat = q.DomainPattern(1.0, np.ones(8, dtype=np.int8))
    with pytest.raises(ValueError, match="process must be 'shg' or 'thg'"):
        q.sweep_spectrum(pat, q.default_dispersion(), [1404.0], "sfg")
    with pytest.raises(ValueError, match="below the model's valid minimum"):
        q.default_dispersion().mismatches_at(100.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_device_spectrum_matches_reference(name):
    import paper_2511_01255_b200 as q

    spec, signs, rows = reference_rows(name)
    pat = q.DomainPattern(spec["thickness"], signs)
    got = q.sweep_spectrum(pat, q.default_dispersion(), rows[:, 0], spec["process"])
    got = np.array(got)
    assert np.array_equal(got[:, 0], rows[:, 0])
    np.testing.assert_allclose(got[:, 1], rows[:, 1], rtol=RTOL)
    np.testing.assert_allclose(got[:, 2], rows[:, 2], rtol=RTOL)


@pytest.mark.gpu
def test_device_spectra_batched_equal_single():
    """Many patterns x many wavelengths in one launch = the per-pattern sweeps."""
    import paper_2511_01255_b200 as q

    rng = np.random.default_rng(3)
    signs = np.where(rng.random((7, 2000)) < 0.5, -1, 1).astype(np.int8)
    wls = np.linspace(1300.0, 1650.0, 97)
    for process in ("thg", "shg"):
        batch = q.sweep_spectra(signs, 0.8, q.default_dispersion(), wls, process)
        assert batch.shape == (7, 97)
        for p in (0, 6):
            one = np.array(q.sweep_spectrum(q.DomainPattern(0.8, signs[p]), q.default_dispersion(), wls, process))
            assert np.array_equal(batch[p], one[:, 1])


@pytest.mark.gpu
@pytest.mark.parametrize("process", ["thg", "shg"])
@pytest.mark.parametrize("temperature", [25.0, 81.5])
def test_device_wavelength_scalars_match_host(process, temperature):
    """Sellmeier dispersion and the moment integrals on the device
    (qpm_wavelength_scalars) against the host formulas the reference uses:
    the mismatches bit-identical, w and the cascade factor within 1e-14."""
    import paper_2511_01255_b200 as q
    from paper_2511_01255_b200.spectrum import _device_wavelength_scalars, _wavelength_scalars

    model = q.default_dispersion(temperature)
    wls = np.concatenate([np.linspace(1250.0, 4900.0, 997), [1404.0, 1380.0, 1430.0]])
    for t in (1.0, 0.37, 25.0):  # series and closed-form branches of the moment integrals
        dk_d, w_d, h_d = _device_wavelength_scalars(model, wls, t, process)
        dk_h, w_h, h_h = _wavelength_scalars(model, wls, t, process)
        assert np.array_equal(dk_d, dk_h)
        np.testing.assert_allclose(w_d, w_h, rtol=1e-14, atol=1e-14 * np.abs(w_h).max())
        np.testing.assert_allclose(h_d, h_h, rtol=1e-14, atol=1e-14 * max(np.abs(h_h).max(), 1e-300))


@pytest.mark.gpu
def test_device_wavelength_scalars_errors_and_tables():
    import paper_2511_01255_b200 as q

    pat = q.DomainPattern(1.0, np.where(np.arange(64) % 3 == 0, -1, 1).astype(np.int8))
    with pytest.raises(ValueError, match="below the model's valid minimum"):
        q.sweep_spectrum(pat, q.default_dispersion(), [1404.0, 1100.0], "thg")  # 1100/3 nm is out of range
    with pytest.raises(ValueError, match="above the model's valid maximum"):
        q.sweep_spectrum(pat, q.default_dispersion(), [6000.0], "shg")
    # an explicit mismatch table keeps the host path and agrees with the model at its own values
    model = q.default_dispersion()
    wls = [1380.0, 1404.0, 1430.0]
    table = q.MismatchTable({w: model.mismatches_at(w) for w in wls})
    a = np.array(q.sweep_spectrum(pat, model, wls, "thg"))
    b = np.array(q.sweep_spectrum(pat, table, wls, "thg"))
    np.testing.assert_allclose(a, b, rtol=1e-13)


@pytest.mark.parametrize("temperature", [25.0, 81.5, -10.0])
def test_sellmeier_terms_restate_the_host_index(temperature):
    """The wavelength-free terms the device receives (_sellmeier_terms) finish
    n(lambda) bit-identically to tables.refractive_index (CPU check of the
    device formula's arithmetic order)."""
    from paper_2511_01255_b200.spectrum import _sellmeier_terms

    model = T.default_dispersion(temperature)
    sm = _sellmeier_terms(model)
    for wl in np.linspace(0.41, 4.99, 501):
        w2 = wl * wl
        n2 = sm[0] - sm[1] * w2
        if sm[2] != 0.0:
            n2 += sm[2] / (w2 - sm[3])
        if sm[4] != 0.0:
            n2 += sm[4] / (w2 - sm[5])
        assert float(np.sqrt(n2)) == T.refractive_index(model, float(wl))


def test_schedule_tables_memoised_read_only():
    from paper_2511_01255_b200 import optimizer as opt

    a = opt._schedule_cached(30, opt.DEParams(), opt.GWOParams(), opt.Schedules())
    b = opt._schedule_cached(30, opt.DEParams(), opt.GWOParams(), opt.Schedules())
    c = opt._schedule_cached(30, opt.DEParams(f_max=0.2), opt.GWOParams(), opt.Schedules())
    assert a is b and c is not a and not a.flags.writeable
    assert np.array_equal(a, opt.schedule_table(30, opt.DEParams(), opt.GWOParams(), opt.Schedules()))
