"""Build libqm.so in-tree for sm_100a (nvcc + g++), no JIT.

    python -m paper_0901_0638_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
ROOT = HERE.parent
LIB = HERE / "libqm.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.cpp")) +
                  list(CSRC.glob("*.h")) + [ROOT / "include" / "qm.h"])


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(s.stat().st_mtime <= t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: Path = None, defines=()) -> Path:
    """`out`/`defines`: an A/B build of the same sources (experiments only)."""
    if out is None and not force and up_to_date():
        return LIB
    lib = LIB if out is None else Path(out)
    # host-side parameter setup (C++, long double / __float128)
    objs = []
    for src in sorted(CSRC.glob("*.cpp")):
        obj = HERE / (src.stem + ".o")
        subprocess.run(["g++", "-O2", "-std=gnu++17", "-fext-numeric-literals", "-fPIC", "-c", str(src),
                        "-o", str(obj)], check=True)
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", str(ROOT / "include"), str(CSRC / "qm_lib.cu"), *map(str, objs), "-lquadmath",
           *[f"-D{d}" for d in defines], "-o", str(lib)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    for o in objs:
        o.unlink(missing_ok=True)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
