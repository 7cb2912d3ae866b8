"""Build the sm_100a shared library in-tree (nvcc; no GPU needed to compile).

    python -m paper_2511_01255_b200.build

The library lands next to this file (paper_2511_01255_b200/libqpm_b200.so),
so it ships to the GPU box with the repo snapshot.  -fmad=false keeps every
multiply and add separately rounded (the reference's arithmetic); kernels
that want FMAs call fma() explicitly.
"""

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqpm_b200.so")
# the same sources with the per-generation invariant checks (-DQPM_CHECKS=1,
# k_check_state); loaded only by tests/test_gpu_checks.py through QPM_LIB
LIB_CHECKS = os.path.join(HERE, "libqpm_b200_checks.so")
SOURCES = ["qpm_fitness.cu", "qpm_engine.cu"]
HEADERS = ["qpm_common.cuh", "qpm_internal.cuh", "qpm_finish.cuh", os.path.join("..", "..", "include", "qpm_b200.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC", "-shared",
              "-cudart", "static", "-Xptxas", "-v"]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build libqpm_b200.so")
    return path


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, checks: bool = False) -> str:
    lib = LIB_CHECKS if checks else LIB
    if not force and not _stale(lib):
        return lib
    tmp = lib + ".tmp"
    extra = os.environ.get("QPM_NVCC_EXTRA", "").split()  # tuning builds, e.g. -DQPM_DE_MINB=3
    if checks:
        extra = extra + ["-DQPM_CHECKS=1"]
    cmd = [nvcc()] + NVCC_FLAGS + extra + ARCH + ["-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, lib)
    if not checks:
        log = os.path.join(HERE, "csrc", "ptxas.log")
        with open(log, "w") as fh:
            fh.write(res.stderr)
    if verbose:
        print(res.stderr, file=sys.stderr)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--checks" in sys.argv:
        print(build(force="--force" in sys.argv, checks=True))
