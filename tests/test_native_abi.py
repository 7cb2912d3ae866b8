"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/qpm_b200.h declares (no compute calls here)."""

import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2511_01255_b200 import _native

HEADER = os.path.join(ROOT, "include", "qpm_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qpm_[a-z0-9_]+)\s*\(", text)))


def test_library_present_and_loads():
    assert os.path.exists(_native.LIB_PATH), "run __graft_entry__.build() first"
    L = _native.lib()
    assert L.qpm_version() >= 10000


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 20
    L = _native.lib()
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(_native.EXPORTS)


def test_compiled_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_host_fold_key_matches_python():
    import ctypes

    import numpy as np

    from paper_2511_01255_b200 import rng

    L = _native.lib()
    for seed, path in ((7, (0, 3)), (-17, (2,)), ((1 << 63) + 5, (1, 2)), (0, ())):
        arr = np.array([rng.signed64(p) for p in path], dtype=np.int64)
        got = L.qpm_fold_key(rng.signed64(seed), len(path), arr.ctypes.data if len(path) else None)
        assert got == rng.fold_key(seed, *path)
    del ctypes


def test_no_cpu_fallback_without_gpu():
    from conftest import has_gpu

    if has_gpu():
        pytest.skip("GPU present")
    import paper_2511_01255_b200 as q

    with pytest.raises(_native.QpmError, match="no CUDA device"):
        q.make_objective(q.ObjectiveSpec("single_thg", (1404.0,)),
                         q.MismatchTable({1404.0: q.PhaseMismatchPair(0.3, 0.7)}), 1.0, 16)


def test_run_params_layout_matches_header(tmp_path):
    """ctypes' RunParams mirrors qpm_run_params field for field (size and offsets
    from the C compiler), so the Python side cannot drift from the ABI."""
    import ctypes

    fields = [name for name, _ in _native.RunParams._fields_]
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "qpm_b200.h"\nint main(void) {\n'
                   '  printf("%zu\\n", sizeof(qpm_run_params));\n'
                   + "".join(f'  printf("%zu\\n", offsetof(qpm_run_params, {f}));\n' for f in fields)
                   + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    res = subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                         capture_output=True, text=True)
    if res.returncode != 0:
        pytest.skip(f"gcc unavailable: {res.stderr[:200]}")
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(_native.RunParams)
    assert vals[1:] == [getattr(_native.RunParams, f).offset for f in fields]
