"""Counter-based random streams (the reference's rng.py API, device-filled).

Stream keys are folded from an integer path (seed, generation, individual)
with splitmix64 exactly as the reference does (rng.py:24-36); value i of a
stream depends only on (key, i), so any span can be regenerated on the device
(_kernels.py:87-98).  Key folding is a few integer ops and stays on the host;
`uniforms` fills on the GPU through qpm_uniform_fill.
"""

import numpy as np

from . import _native

MASK64 = (1 << 64) - 1
GOLD = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return (z ^ (z >> 31)) & MASK64


def fold_key(seed: int, *path: int) -> int:
    h = _mix(seed & MASK64)
    for p in path:
        h = _mix(h + GOLD + (p & MASK64))
    return h


def signed64(x: int) -> int:
    x &= MASK64
    return x - (1 << 64) if x >= (1 << 63) else x


def uniform_fill_device(key: int, start: int, n: int, out=None, stream=None):
    """n doubles of stream `key` from position `start` into a CUDA tensor."""
    import torch

    dev = _native.require_cuda()
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=dev)
    _native.check(_native.lib().qpm_uniform_fill(key & MASK64, start, n, out.data_ptr(),
                                                 _native.stream_handle(stream)), "qpm_uniform_fill")
    return out


def uniform_fill(key: int, start: int, n: int) -> np.ndarray:
    """Host copy of a device fill (the reference's _kernels.uniform_fill contract)."""
    if n == 0:
        return np.empty(0, dtype=np.float64)
    return uniform_fill_device(key, start, n).cpu().numpy()


class CounterStream:
    """Sequential view over one keyed stream; the position is the only state."""

    __slots__ = ("key", "_pos")

    def __init__(self, seed: int, *path: int):
        self.key = fold_key(seed, *path)
        self._pos = 0

    def uniforms(self, n: int) -> np.ndarray:
        out = uniform_fill(self.key, self._pos, n)
        self._pos += n
        return out

    def uniform(self) -> float:
        return float(self.uniforms(1)[0])

    def randint(self, bound: int) -> int:
        return min(int(self.uniform() * bound), bound - 1)

    def randints(self, n: int, bound: int) -> np.ndarray:
        u = self.uniforms(n)
        return np.minimum((u * bound).astype(np.int64), bound - 1)


def stream(seed: int, *path: int) -> CounterStream:
    return CounterStream(seed, *path)


def random_population_matrix(rows: int, n: int, seed: int = 0) -> np.ndarray:
    """bench.random_population_matrix (bench.py:216-218): +/-1 with p = 1/2."""
    u = uniform_fill(fold_key(seed, 0), 0, rows * n)
    return np.where(u < 0.5, -1, 1).astype(np.int8).reshape(rows, n)
