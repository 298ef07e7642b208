"""Build libelas.so in-tree (nvcc, sm_100a only) and the C oracle helpers (none yet).

Usage: python -m paper_2601_08374_b200.build   (or __graft_entry__.build()).
Compiles each translation unit in parallel, links one shared library with NCCL.
"""

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, os.environ.get("ELAS_LIBNAME", "libelas.so"))
EXTRA = [f"-D{d}" for d in os.environ.get("ELAS_DEFINES", "").split()]
DEBUG_LIB = "libelas_debug.so"   # ELAS_DEBUG=1: device bounds checks (elas_debug_checks)
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
              "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _nccl_paths():
    try:
        import nvidia.nccl as n
        base = list(n.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _digest():
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(name.encode() + f.read())
    with open(os.path.join(INCLUDE, "elas.h"), "rb") as f:
        h.update(f.read())
    h.update(" ".join(ARCH + NVCC_FLAGS + EXTRA).encode())
    return h.hexdigest()[:16]


def _compile(src, obj, nccl_inc):
    cmd = ["nvcc", *ARCH, *NVCC_FLAGS, *EXTRA, "-I", INCLUDE, "-I", nccl_inc, "-c",
           os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return src, r.stderr


def build(force=False, verbose=False, debug=False):
    """Compile every CUDA/C++ source for sm_100a and link lib/libelas.so (skips if up to date).
    debug=True: lib/libelas_debug.so with ELAS_DEBUG=1 (device bounds checks)."""
    global LIB, EXTRA
    if debug:
        saved = LIB, EXTRA
        LIB, EXTRA = os.path.join(LIBDIR, DEBUG_LIB), EXTRA + ["-DELAS_DEBUG=1"]
        try:
            return _build(force, verbose, "obj" + DEBUG_LIB)
        finally:
            LIB, EXTRA = saved
    return _build(force, verbose, "obj" + os.environ.get("ELAS_LIBNAME", ""))


def _build(force, verbose, objname):
    os.makedirs(LIBDIR, exist_ok=True)
    stamp = LIB + ".stamp"
    dig = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == dig:
                return LIB
    nccl_inc, nccl_lib = _nccl_paths()
    objdir = os.path.join(LIBDIR, objname)
    os.makedirs(objdir, exist_ok=True)
    srcs = _sources()
    objs = [os.path.join(objdir, s.rsplit(".", 1)[0] + ".o") for s in srcs]
    logs = {}
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        futs = [ex.submit(_compile, s, o, nccl_inc) for s, o in zip(srcs, objs)]
        for f in cf.as_completed(futs):
            src, log = f.result()
            logs[src] = log
    with open(LIB + ".ptxas.log", "w") as f:
        for src in sorted(logs):
            f.write(f"== {src}\n{logs[src]}\n")
    tmp = LIB + ".tmp"
    cmd = ["nvcc", *ARCH, "-shared", "-o", tmp, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath={nccl_lib}", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(dig)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv)
