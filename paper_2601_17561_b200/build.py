"""In-tree build of the B200 engine: nvcc for sm_100a -> libirl_b200.so.

    python -m paper_2601_17561_b200.build [--debug]

The shared library is written next to this file so it ships with the repo
snapshot to the GPU box. Objects go to build/ at the repo root.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
OUT = PKG / "libirl_b200.so"
BUILD = ROOT / "build"

CUDA_SOURCES = ["ppmm_gemm.cu", "kernels_aux.cu", "capi.cu", "ccmm_engine.cu", "ccmm_group.cu", "iris.cu", "fold.cu"]
HOST_SOURCES = ["modmat_b200.cpp", "iris_b200.cpp", "ccmm_b200.cpp"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _host_cxx() -> str:
    # /usr/bin/g++ links the shared libstdc++ the Python process already uses.
    return "/usr/bin/g++" if Path("/usr/bin/g++").exists() else (shutil.which("g++") or "g++")


def _compile(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stderr


def build(debug: bool = False, verbose: bool = False, defines=(), out: Path = OUT) -> Path:
    """defines / out: experiment variants (e.g. -DIRL_EPI_WARPS=8 into build/variants/),
    loaded with IRL_B200_LIB=<path>; the product library is always OUT."""
    out = Path(out)
    bdir = BUILD if out == OUT else out.parent / (out.stem + ".obj")
    bdir.mkdir(parents=True, exist_ok=True)
    nvcc = _nvcc()
    cxx = _host_cxx()
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-ccbin", cxx,
              f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{HOST}"]
    if debug:
        common.append("-DIRL_WAIT_TIMEOUT")
    common += [f"-D{d}" for d in defines]
    jobs = []
    objs = []
    for src in CUDA_SOURCES:
        obj = bdir / (Path(src).stem + ".o")
        objs.append(obj)
        jobs.append([nvcc, *ARCH, *common, "-Xptxas", "-v", "-c", str(CSRC / src), "-o", str(obj)])
    for src in HOST_SOURCES:
        if not (HOST / src).exists():
            continue
        obj = bdir / (Path(src).stem + ".o")
        objs.append(obj)
        jobs.append([cxx, "-O2", "-std=c++17", "-fPIC", f"-I{ROOT / 'include'}", f"-I{HOST}",
                     "-I/usr/local/cuda/include", "-c", str(HOST / src), "-o", str(obj)])
    with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        logs = list(ex.map(_compile, jobs))
    if verbose:
        for log in logs:
            sys.stderr.write(log)
    link = [nvcc, *ARCH, "-shared", "-ccbin", cxx, "-o", str(out), *map(str, objs), "-lcudart_static",
            "-lrt", "-ldl", "-lpthread"]
    _compile(link)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--debug", action="store_true", help="trap on stuck mbarrier waits")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="experiment define")
    ap.add_argument("--out", default=str(OUT), help="variant library path (load with IRL_B200_LIB)")
    a = ap.parse_args()
    print(build(debug=a.debug, verbose=a.verbose, defines=a.defines, out=Path(a.out)))


if __name__ == "__main__":
    main()
