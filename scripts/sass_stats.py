"""Static SASS statistics of one kernel (no GPU): compile a csrc/*.cu file to a
cubin for sm_100a and count opcodes of the kernels whose mangled name matches.

    python scripts/sass_stats.py px_tb.cu k_tb ILi0ELi4ELi15ELi1ELi0E
"""
import collections
import os
import re
import subprocess
import sys

import importlib.util

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2307_07931_b200", "csrc")


def main():
    src, *pats = sys.argv[1:]
    spec = importlib.util.find_spec("nvidia.nccl")
    nccl = list(spec.submodule_search_locations)[0]
    out = f"/tmp/sass_{os.path.basename(src)}.cubin"
    subprocess.run(["nvcc", "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-cubin", f"-I{ROOT}/include", f"-I{CSRC}", f"-I{nccl}/include", "-Xptxas", "-v",
                    os.path.join(CSRC, src), "-o", out], check=True)
    sass = subprocess.run(["cuobjdump", "-sass", out], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if not all(p in name for p in pats):
            continue
        ops = collections.Counter()
        for line in f.split("\n"):
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                ops[m.group(2)] += 1
        print(name, sum(ops.values()))
        print("  ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(40)))


if __name__ == "__main__":
    main()
