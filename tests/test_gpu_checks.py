"""GPU: the engine's invariant checks (compute-sanitizer is not available on
this pool, so the engine carries its own asserts).

libqpm_b200_checks.so is the same sources built with -DQPM_CHECKS=1: after
every generation k_check_state verifies that slot_of/spare_of stay a
permutation of the 2 NP slots, that the planner's next DE picks are distinct,
!= i and in range with a valid j_rand, that the leaders are distinct and in
range, that every fitness and the new trace row are finite, and that the
planner's generation counter is in step.  Eight configurations (C2 shape,
planner fork at the start with wolf planes on the side stream -- the round-1
schedule that gave run-to-run differences --, the side-stream wolf
placement, 3 leaders, DE, GWO, NP > 4096 with multi-CTA selection, several
wavelengths) must raise no flag and give the same traces as the normal
library (the checks only read).
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2511_01255_b200")


def run_worker(lib):
    env = dict(os.environ, QPM_LIB=lib)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "checks_worker.py")], capture_output=True,
                         text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-3000:]
    return json.loads(res.stdout.strip().splitlines()[-1])


def test_invariant_checks_clean_and_inert():
    checked = os.path.join(PKG, "libqpm_b200_checks.so")
    assert os.path.exists(checked), "build it with __graft_entry__.build() (paper_2511_01255_b200.build --checks)"
    got = run_worker(checked)
    plain = run_worker(os.path.join(PKG, "libqpm_b200.so"))
    for g, p in zip(got, plain):
        assert g["checks"], g
        assert g["flags"] == 0, f"run {g['run']}: invariant violation flags {g['flags']:#x} detail {g['detail']:#x}"
        assert not p["checks"]  # the product library has no check state
        assert g["digest"] == p["digest"], f"run {g['run']}: the checks changed the trace"
