"""Build libqcb200.so (sm_100a) in-tree with nvcc.

    python -m paper_2306_12063_b200._build [--verbose] [--force]

Each csrc/*.cu is compiled to an object in parallel
(`-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`, no fast-math: the
decoder's float path must stay IEEE-exact), then linked into
`paper_2306_12063_b200/libqcb200.so`.  The .so is git-ignored but travels to
the GPU box with the gpurun snapshot.
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
CSRC = PKG / "csrc"
OBJ = PKG / os.environ.get("QCB_BUILD_DIR", "build")
LIB = Path(os.environ.get("QCB_LIB") or PKG / "libqcb200.so")
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-I", str(CSRC), "-I", str(INCLUDE)]
EXTRA = os.environ.get("QCB_NVCC_EXTRA", "").split()   # tuning experiments only


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    src = sorted(CSRC.glob("*.cu"))
    if "-DQCB_SCALED_KERNELS=0" in EXTRA:          # experiment builds: no per-Z scaled decoders
        src = [s for s in src if not s.name.startswith("dec_scaled_")]
    return src


def _deps():
    return sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [INCLUDE / "qcb200.h"]


def _stale(target: Path, inputs) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(p.stat().st_mtime > t for p in inputs)


def _compile(src: Path, verbose: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    cmd = [nvcc(), *NVCC_FLAGS, *EXTRA, "-c", str(src), "-o", str(obj)]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
    if verbose and (res.stdout or res.stderr):
        sys.stderr.write(res.stderr + res.stdout)
    return obj


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    deps = _deps()
    todo = [s for s in _sources() if force or _stale(OBJ / (s.stem + ".o"), [s, *deps])]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            list(ex.map(lambda s: _compile(s, verbose), todo))
    objs = [OBJ / (s.stem + ".o") for s in _sources()]
    if force or todo or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart"]
        subprocess.run(cmd, check=True, capture_output=not verbose)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args()
    print(build(verbose=args.verbose, force=args.force))
