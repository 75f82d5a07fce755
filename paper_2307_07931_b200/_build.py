"""Build libprotox.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery): the .so travels to the GPU box with the repo."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libprotox.so")
INCLUDE = os.path.join(ROOT, "include")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("NCCL headers/library (nvidia.nccl) not found")
    return list(spec.submodule_search_locations)[0]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "protox.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every source to an object in parallel (one nvcc per file), then
    link libprotox.so.  Objects are cached in build/ under a hash of the
    source, every header and the command line (force=True recompiles all)."""
    if not force and not needs_build():
        return LIB
    import concurrent.futures as cf
    import hashlib
    nccl = nccl_dir()
    common = ["nvcc", "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
              f"-I{INCLUDE}", f"-I{CSRC}", f"-I{nccl}/include"]
    odir = os.path.join(PKG, "build")
    os.makedirs(odir, exist_ok=True)
    log = os.path.join(PKG, "build.log")
    hdrs = b"".join(open(h, "rb").read() for h in sorted(glob.glob(os.path.join(CSRC, "*.h")) +
                                                         glob.glob(os.path.join(CSRC, "*.cuh")) +
                                                         [os.path.join(INCLUDE, "protox.h")]))
    tmp = None
    try:
        def compile_one(src):
            key = hashlib.sha1(open(src, "rb").read() + hdrs + " ".join(common).encode()).hexdigest()[:16]
            base = os.path.basename(src)
            obj = os.path.join(odir, f"{base}.{key}.o")
            cmd = [*common, "-Xptxas", "-v", "-c", src, "-o", obj + ".part"]
            if os.path.exists(obj) and not force:
                return src, obj, cmd, subprocess.CompletedProcess(cmd, 0, "(cached)\n", "")
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode == 0:
                os.replace(obj + ".part", obj)
                for old in glob.glob(os.path.join(odir, f"{base}.*.o")):
                    if old != obj:
                        os.remove(old)
            return src, obj, cmd, r
        srcs = sources()
        with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
            results = list(ex.map(compile_one, srcs))
        text = []
        failed = []
        for src, obj, cmd, r in results:
            text.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                failed.append((src, r.stderr))
        if not failed:
            tmp = LIB + f".tmp{os.getpid()}"
            cmd = ["nvcc", *ARCH, "-shared", *[o for _, o, _, _ in results], f"-L{nccl}/lib", "-l:libnccl.so.2",
                   f"-Xlinker=-rpath,{nccl}/lib", "-o", tmp]
            r = subprocess.run(cmd, capture_output=True, text=True)
            text.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                failed.append(("link", r.stderr))
        with open(log, "w") as f:
            f.write("\n".join(text))
        if failed:
            for src, err in failed:
                sys.stderr.write(f"--- {src}\n{err[-6000:]}\n")
            raise RuntimeError(f"nvcc failed (see {log})")
        os.replace(tmp, LIB)
    finally:
        if tmp and os.path.exists(tmp):
            os.remove(tmp)
    if verbose:
        with open(log) as f:
            print(f.read())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
