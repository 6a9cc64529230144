"""Builds libmpwsd.so in-tree with nvcc for sm_100a (no JIT cache, so the
built library travels with the repo snapshot to the GPU box).  Each
translation unit compiles in its own nvcc process (in parallel), then one
link step produces the shared library."""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(CSRC, "build")
LIB = os.path.join(HERE, "libmpwsd.so")
PROF_LIB = os.path.join(HERE, "libmpwsd_prof.so")
SOURCES = ["mpwsd.cu", "hop_tc.cu", "hop_ar.cu", "scl_lane.cu", "sphere_tools.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*os.environ.get("MPW_EXTRA_CFLAGS", "").split(), *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"]


def _deps():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)
            if f.endswith((".cu", ".cuh", ".h", ".cpp"))]
    deps.append(os.path.join(HERE, "..", "include", "mpwsd.h"))
    return deps


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps() if os.path.exists(d))


def _obj(src: str, obj_dir: str = OBJ) -> str:
    return os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")


def _obj_stale(src: str, obj_dir: str = OBJ) -> bool:
    """An object is stale when it or its dependency file is missing, or any
    file the dependency file lists (nvcc -MD) is newer."""
    o, d = _obj(src, obj_dir), _obj(src, obj_dir)[:-2] + ".d"
    if not (os.path.exists(o) and os.path.exists(d)):
        return True
    t = os.path.getmtime(o)
    with open(d) as fh:
        deps = fh.read().replace("\\\n", " ").split(":", 1)[-1].split()
    return any(not os.path.exists(f) or os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False, profile: bool = False) -> str:
    """profile=True: the profiling library (-DMPW_PROFILE: per-tile clock
    trace of the hop kernel) as libmpwsd_prof.so, selected with MPW_LIB."""
    lib, obj_dir = (PROF_LIB, OBJ + "_prof") if profile else (LIB, OBJ)
    if not force and not profile and not _stale():
        return LIB
    os.makedirs(obj_dir, exist_ok=True)
    extra = ["-Xptxas=-v"] if verbose else []
    if profile:
        extra.append("-DMPW_PROFILE")
    todo = [s for s in SOURCES if force or _obj_stale(s, obj_dir)]

    def compile_one(src):
        cmd = [NVCC, *CFLAGS, *extra, "-MD", "-MF", _obj(src, obj_dir)[:-2] + ".d", "-c", os.path.join(CSRC, src),
               "-o", _obj(src, obj_dir)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
        return src, r

    with ThreadPoolExecutor(max_workers=max(1, len(todo))) as ex:
        results = list(ex.map(compile_one, todo))
    for src, r in results:
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, f"nvcc {src}")
    cmd = [NVCC, *ARCH, "-shared", "-o", lib + ".tmp", *[_obj(s, obj_dir) for s in SOURCES], "-lpthread"]
    subprocess.run(cmd, check=True, cwd=HERE)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, profile="--profile" in sys.argv))
