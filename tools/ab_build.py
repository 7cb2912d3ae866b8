"""Build A/B variants of libqpm_b200.so with extra nvcc defines (here, no GPU needed).

    python tools/ab_build.py NAME='-DQPM_XS30=0 -DQPM_XS27=0' NAME2='...'
Each lands in build/ab/libqpm_<NAME>.so; time them on the GPU with tools/ab_run.sh.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_01255_b200 import build as b  # noqa: E402

OUT = os.path.join(os.path.dirname(b.HERE), "build", "ab")


def main():
    os.makedirs(OUT, exist_ok=True)
    for arg in sys.argv[1:]:
        name, _, flags = arg.partition("=")
        lib = os.path.join(OUT, f"libqpm_{name}.so")
        cmd = [b.nvcc()] + b.NVCC_FLAGS + flags.split() + b.ARCH + ["-o", lib] + \
            [os.path.join(b.CSRC, s) for s in b.SOURCES]
        res = subprocess.run(cmd, cwd=b.CSRC, capture_output=True, text=True)
        if res.returncode:
            sys.exit(res.stderr)
        spill = [ln for ln in res.stderr.splitlines() if "spill" in ln]
        regs = [ln for ln in res.stderr.splitlines() if "Used" in ln]
        i = [k for k, ln in enumerate(res.stderr.splitlines()) if "k_de_trialILi4" in ln and "Compiling" in ln]
        lines = res.stderr.splitlines()
        info = " | ".join(lines[i[0] + 1:i[0] + 4]) if i else ""
        print(name, lib, info[:300], len(spill), len(regs))


if __name__ == "__main__":
    main()
