"""Exhaustive search on the device (drop-in for bench.brute_force_oracle).

Mirrors /root/reference/pkg/src/qpmdesign/bench.py:165-209: pattern number
`index` has sign j = -1 iff bit n-1-j of the index is set, so index 0 is the
all-up pattern and the enumeration is lexicographic with +1 before -1; the
optimum's ties go to the lexicographically first pattern.  The patterns are
generated, scored and reduced on the B200 (`qpm_brute_force`), chunk_rows at a
time.  The reference refuses n > 20; `limit` keeps that default and lets a
caller lift it (2^n evaluations).
"""

import ctypes

import numpy as np

from . import _native

ORACLE_LIMIT = 20  # bench._ORACLE_LIMIT


def lexicographic_signs(index: int, n: int) -> np.ndarray:
    """Pattern number `index` in the documented order: +1 sorts before -1 (bench.py:169-176)."""
    bits = (index >> np.arange(n - 1, -1, -1)) & 1
    return (1 - 2 * bits).astype(np.int8)


def brute_force_oracle(objective, n: int, chunk: int = 1 << 20, limit: int = ORACLE_LIMIT,
                       mode: str | None = None) -> tuple[np.ndarray, float]:
    """Global optimum over all 2^n sign patterns of a GpuPatternObjective with dimension n."""
    if n < 1:
        raise ValueError(f"n must be >= 1, got {n}")
    if n > limit:
        raise ValueError(
            f"n={n} needs 2^{n} = {2 ** n} evaluations; the exhaustive oracle refuses n > {limit}"
        )
    if getattr(objective, "dimension", n) != n:
        raise ValueError(f"n={n} does not match the objective's dimension {objective.dimension}")
    from .objectives import MODES

    idx = ctypes.c_int64()
    fit = ctypes.c_double()
    lib = _native.lib()
    m = MODES[mode or objective.mode]
    _native.check(lib.qpm_brute_force(objective.handle, int(n), m, int(chunk), ctypes.byref(idx), ctypes.byref(fit),
                                      None), "qpm_brute_force")
    return lexicographic_signs(int(idx.value), n), float(fit.value)
