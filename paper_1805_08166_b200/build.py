"""Build libautotvm_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1805_08166_b200.build [--force] [--verbose]

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false.
-fmad=false keeps every fp32/fp64 a*b+c as two IEEE RN operations (the oracle is
compiled with -ffp-contract=off); FMAs that the method wants are explicit
__fmaf_rn calls.  No --use_fast_math: IEEE division / sqrt, denormals kept.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libautotvm_b200.so"
OBJ = ROOT / "build" / "obj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["runtime.cu", "space.cu", "features.cu", "gbt.cu", "sa.cu", "topk.cu", "select.cu", "fit.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include"), "-Xptxas", "-warn-spills"]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), lib: Path = None) -> Path:
    """defines: extra -D flags for an instrumented variant (e.g. AT_SA_PHASE_TIMING), built into its own
    object directory and `lib` path (tools only; the product library is the default build)."""
    lib = LIB if lib is None else Path(lib)
    obj = OBJ if not defines else OBJ.parent / ("obj_" + "_".join(d.lstrip("-D").lower() for d in defines))
    obj.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "at_b200.h"]
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = obj / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers, Path(__file__)]):
            cmd = [NVCC, *FLAGS, *defines, "-c", str(s), "-o", str(o)]
            if verbose:
                cmd += ["-Xptxas", "-v"]
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or _stale(lib, objs):
        tmp = lib.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp),
                               *map(str, objs), "-lcudart_static", "-lrt", "-ldl", "-lpthread"])
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
