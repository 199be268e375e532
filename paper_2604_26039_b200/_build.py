"""Builds libramp_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2604_26039_b200._build      # or __graft_entry__.build()

The library is the C ABI of include/ramp_b200.h; it depends only on the
CUDA runtime (the driver's tensor-map encoder is fetched at run time through
cudaGetDriverEntryPointByVersion, so no -lcuda is needed to link).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_objs"
LIB = PKG / "libramp_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-v"]
# The route TU evaluates the fp64 cost model; -fmad=false keeps every product
# and sum separately rounded, matching numpy's evaluation (ramp/cost_model.py:114).
PER_FILE = {"route.cu": ["-fmad=false"]}
SOURCES = ["route.cu", "moe.cu", "ep.cu", "capi.cu"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    # development builds (timeline probes): RAMP_EXTRA_NVCC="-DRAMP_START_STAMPS" etc.
    extra = os.environ.get("RAMP_EXTRA_NVCC", "").split()
    headers = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [PKG.parent / "include" / "ramp_b200.h"]
    objs = []
    for src in SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [CSRC / src, *headers]):
            cmd = [nvcc(), *ARCH, *COMMON, *extra, *PER_FILE.get(src, []), "-c", str(CSRC / src), "-o", str(obj)]
            res = subprocess.run(cmd, capture_output=True, text=True)
            log = BUILD / (Path(src).stem + ".ptxas.log")
            log.write_text(res.stdout + res.stderr)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                print(res.stderr)
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link of libramp_b200.so failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
