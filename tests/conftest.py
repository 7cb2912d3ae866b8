"""Shared pytest setup: the `gpu` marker, golden-fixture loaders, repo paths.

CPU tests (`-m "not gpu"`) cover the oracle against the reference's golden
vectors, the host-side mirror of the reference API, and that the C-ABI library
loads and exports every declared symbol.  GPU tests (`-m gpu`) are the parity
tests proper: they call the CUDA engine through the C-ABI and compare with the
oracle and the golden vectors.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


_CACHE = {}


def golden(name: str):
    if name not in _CACHE:
        _CACHE[name] = dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))
    return _CACHE[name]


def unpack_signs(packed: np.ndarray, n: int) -> np.ndarray:
    bits = np.unpackbits(packed, axis=-1, count=n, bitorder="little")
    return (1 - 2 * bits.astype(np.int8)).astype(np.int8)


def spec_of(fix, name):
    return json.loads(str(fix[f"{name}__spec"]))
