"""Build libf4b200.so in-tree (nvcc, sm_100a).

Every ``csrc/*.cu`` is compiled to an object in parallel, then linked into
``paper_2601_06765_b200/libf4b200.so``.  Flags: ``-gencode
arch=compute_100a,code=sm_100a -O3 -lineinfo``.  Rebuilds only when a source
or header is newer than the library.  ``csrc/hostglue.cpp`` (host glue of the
F4 driver: compile_batch's row-list packing and the Gebauer-Moeller criteria,
a CPython extension) is compiled with g++ into
``paper_2601_06765_b200/_hostglue*.so``.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libf4b200.so")
OBJ_DIR = os.path.join(ROOT, "build", "obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(ROOT, "include", "f4b200.h"))
    return any(os.path.getmtime(p) > t for p in deps)


HOSTGLUE_SRC = os.path.join(CSRC, "hostglue.cpp")
HOSTGLUE = os.path.join(HERE, "_hostglue" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def build_hostglue(force: bool = False) -> str:
    if not force and os.path.exists(HOSTGLUE) and os.path.getmtime(HOSTGLUE) >= os.path.getmtime(HOSTGLUE_SRC):
        return HOSTGLUE
    tmp = HOSTGLUE + ".tmp"
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-shared", "-fPIC", "-Wall", "-I",
           sysconfig.get_paths()["include"], HOSTGLUE_SRC, "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed for {HOSTGLUE_SRC}:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, HOSTGLUE)
    return HOSTGLUE


def build(force: bool = False, verbose: bool = False, extra=()) -> str:
    build_hostglue(force)
    if not force and not _stale():
        return LIB
    os.makedirs(OBJ_DIR, exist_ok=True)
    nvcc = _nvcc()

    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    hdrs.append(os.path.join(ROOT, "include", "f4b200.h"))
    t_hdr = max(os.path.getmtime(h) for h in hdrs)

    def compile_one(src):
        obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), t_hdr):
            return obj  # object newer than its source and every header
        cmd = [nvcc, *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
        if verbose and (res.stdout.strip() or res.stderr.strip()):
            sys.stderr.write(res.stdout + res.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = LIB + ".tmp"
    cmd = [nvcc, *ARCH, "-shared", "-o", tmp, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
