"""Build libmemshare.so for sm_100a (nvcc; runs without a GPU)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libmemshare.so")
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
              "-shared", "-Xptxas", "-warn-spills"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "memshare.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = ["nvcc", *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-o", OUT, *sources()]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    return OUT


def build_variant(name: str, defines) -> str:
    """Tuning experiments: an extra .so with -D overrides (never the shipped library)."""
    out = os.path.join(HERE, f"libmemshare_{name}.so")
    cmd = ["nvcc", *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I" + os.path.join(ROOT, "include"), "-o", out,
           *sources()]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
