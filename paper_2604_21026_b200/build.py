"""Build libmcapq.so in-tree for sm_100a (nvcc; no torch extension machinery).

    python -m paper_2604_21026_b200.build [--force]

Every .cu/.cpp under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` (no fast-math: the
quantisers must be IEEE-exact) and linked against the venv's NCCL 2.28.  The
ptxas resource report (registers, spills, smem) is written to
``build/ptxas.log``.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import importlib.util
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libmcapq.so"
INCLUDE = PKG.parent / "include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def nccl_dirs():
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    raise RuntimeError("venv NCCL (nvidia/nccl) not found; /usr/include's 2.27 headers do not match torch's 2.28")


def _sources():
    return sorted(glob.glob(str(CSRC / "*.cu")) + glob.glob(str(CSRC / "*.cpp")))


def _headers():
    return sorted(glob.glob(str(CSRC / "*.h")) + glob.glob(str(CSRC / "*.cuh")) + [str(INCLUDE / "mcapq.h")])


def _compile(src: str, nccl_inc: str) -> tuple[str, str]:
    obj = OBJ / (Path(src).name + ".o")
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
           "--expt-relaxed-constexpr", "-I", str(INCLUDE), "-I", nccl_inc, "-c", src, "-o", str(obj)]
    if src.endswith(".cpp"):
        cmd = [nvcc(), "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(INCLUDE), "-I", nccl_inc,
               "-x", "c++", "-c", src, "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return str(obj), r.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    srcs = _sources()
    deps = srcs + _headers() + [__file__]
    if LIB.exists() and not force:
        t = LIB.stat().st_mtime
        if all(os.stat(d).st_mtime <= t for d in deps):
            return LIB
    OBJ.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    nccl_inc, nccl_lib = nccl_dirs()
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        futs = [ex.submit(_compile, s, nccl_inc) for s in srcs]
        objs = []
        for f in futs:
            o, log = f.result()
            objs.append(o)
            logs.append(f"== {Path(o).name}\n{log}")
    (OBJ / "ptxas.log").write_text("\n".join(logs))
    tmp = LIB.with_suffix(f".so.{os.getpid()}.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-L", nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{nccl_lib}", "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
