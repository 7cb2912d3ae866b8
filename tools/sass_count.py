"""Static SASS size of kernels in libqpm_b200.so (offline proxy for instruction-count work).

    python tools/sass_count.py [LIB] [NAME_SUBSTR...]
"""
import collections
import re
import subprocess
import sys


def functions(lib):
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, out = None, collections.OrderedDict()
    for ln in txt.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            out[cur] = []
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(.*?);", ln)
        if cur and m:
            out[cur].append(m.group(1))
    return out


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2511_01255_b200/libqpm_b200.so"
    want = sys.argv[2:] or ["k_de_trialILi4"]
    for name, ins in functions(lib).items():
        if not any(w in name for w in want):
            continue
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0].split(".")[0] for i in ins)
        print(name, len(ins), dict(ops.most_common(12)))


if __name__ == "__main__":
    main()
