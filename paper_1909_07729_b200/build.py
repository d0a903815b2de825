"""Build libktanh.so (sm_100a) in-tree with nvcc.

    python paper_1909_07729_b200/build.py [--force]

(run it as a script: importing the package needs the library it builds)

The library links the CUDA runtime statically, so the .so needs only the
driver at run time; it never links torch.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libktanh.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",                    # no silent FMA contraction in fp32 scaffolding
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-O2",
    "-cudart", "static",
    "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) \
        + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build_variant(out: str, defines: list[str]) -> str:
    """Dev A/B build: the same sources with extra -D flags into `out` (load it
    with KT_LIB=<out>; abtmp/ is git-ignored but travels to the GPU box)."""
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-I", INCLUDE, "-I", CSRC, "-o", out] + sources()
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed")
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = LIB + ".tmp%d" % os.getpid()
    cmd = [nvcc] + NVCC_FLAGS + ["-I", INCLUDE, "-I", CSRC, "-o", tmp] + sources()
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libktanh.so")
    if verbose:
        sys.stderr.write(r.stderr)
    with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:   # registers / spills per kernel
        f.write("".join(ln for ln in r.stderr.splitlines(keepends=True) if "Compile time" not in ln))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    # python build.py [--force] | --variant OUT.so DEF[=V] ...
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
