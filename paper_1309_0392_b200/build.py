"""Build libsgh.so in-tree with nvcc for sm_100a (B200).

    python paper_1309_0392_b200/build.py [--force] [--verbose]

(run it as a script: importing the package loads libsgh.so, which is what
this script produces)

The shared library is written to paper_1309_0392_b200/lib/libsgh.so (git-ignored,
but it travels to the GPU box with the gpurun snapshot).  NCCL comes from the
venv's nvidia-nccl wheel (the same libnccl.so.2 torch loads); the CUDA runtime
is linked statically so the library does not depend on a second libcudart.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(OUT_DIR, "libsgh.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    import nvidia.nccl  # the wheel torch links against (NCCL 2.28)
    base = os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp"))) + [
        os.path.join(ROOT, "include", "sgh.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build LIB (or a tuning variant at `out` with extra -D defines)."""
    target = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    inc, libdir = nccl_paths()
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-cudart", "static", "-Xptxas", "-v" if verbose else "-O3",
           f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}", *[f"-D{d}" for d in defines],
           *sources(), "-o", target + ".tmp",
           f"-L{libdir}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={libdir}"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libsgh.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None, help="build a tuning variant here instead of lib/libsgh.so")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra preprocessor define")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.out, a.defines))
