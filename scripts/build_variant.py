"""Build an A/B variant of libprotox.so: one source recompiled with extra
nvcc flags (e.g. -DPX_RS_DIAG=1), linked with the cached objects of the
others into paper_2307_07931_b200/libprotox_<name>.so (select it with
PROTOX_LIB=...).  Measurement tooling only.

usage: python scripts/build_variant.py NAME SOURCE.cu FLAG...
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2307_07931_b200 import _build as B  # noqa: E402

name, src, flags = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()  # the cached objects of the default build
nccl = B.nccl_dir()
odir = os.path.join(B.PKG, "build")
base = os.path.basename(src)
objs = [o for o in glob.glob(os.path.join(odir, "*.o")) if not os.path.basename(o).startswith(base + ".")]
vobj = os.path.join("/tmp", f"{base}.{name}.o")
cmd = ["nvcc", "-std=c++17", "-O3", "-lineinfo", *B.ARCH, "-Xcompiler", "-fPIC", f"-I{B.INCLUDE}", f"-I{B.CSRC}",
       f"-I{nccl}/include", *flags, "-c", os.path.join(B.CSRC, base), "-o", vobj]
subprocess.run(cmd, check=True)
out = os.path.join(B.PKG, f"libprotox_{name}.so")
subprocess.run(["nvcc", *B.ARCH, "-shared", *objs, vobj, f"-L{nccl}/lib", "-l:libnccl.so.2",
                f"-Xlinker=-rpath,{nccl}/lib", "-o", out], check=True)
print(out)
