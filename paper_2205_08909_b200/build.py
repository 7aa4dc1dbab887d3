"""Build ``libmfcg_b200.so`` in-tree with nvcc for sm_100a.

One translation unit per polynomial degree (``mfcg_inst.cu`` with
``-DMFCG_P=k``) plus the C-ABI unit, compiled in parallel and linked into
``paper_2205_08909_b200/libmfcg_b200.so``.  nvcc cross-compiles without a GPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OBJ = CSRC / "build"
LIB = PKG / "libmfcg_b200.so"
DEGREES = tuple(range(1, 9))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", f"-I{INCLUDE}", f"-I{CSRC}",
]


def _nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found; cannot build libmfcg_b200.so")
    return exe


def _sources():
    return [CSRC / "mfcg_b200.cu", CSRC / "mfcg_inst.cu", CSRC / "mfcg_kernels.cuh",
            CSRC / "mfcg_engine.cuh", CSRC / "mfcg_brick2.cuh", INCLUDE / "mfcg_b200.h"]


def is_stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(src.stat().st_mtime > t for src in _sources())


def _compile(args):
    src, obj, extra = args
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-c", str(src), "-o", str(obj)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    return obj


def build_variant(out: Path, flags, degrees=DEGREES, verbose: bool = False) -> Path:
    """A variant build (extra -D flags) into its own file and object directory; load it with MFCG_LIB=<out>."""
    out = Path(out)
    objdir = OBJ / ("var_" + out.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    jobs = [(CSRC / "mfcg_b200.cu", objdir / "mfcg_b200.o", list(flags))]
    jobs += [(CSRC / "mfcg_inst.cu", objdir / f"mfcg_inst_p{p}.o",
              [f"-DMFCG_P={p}", *flags] if p in degrees else [f"-DMFCG_P={p}", "-DMFCG_STUB"]) for p in DEGREES]
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as pool:
        objs = list(pool.map(_compile, jobs))
    cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(out), *map(str, objs)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    if verbose:
        print(f"built {out}", file=sys.stderr)
    return out


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile and link the shared library if it is missing or out of date."""
    if os.environ.get("MFCG_EXTRA_FLAGS"):
        raise RuntimeError("MFCG_EXTRA_FLAGS would change the production library: use build_variant() + MFCG_LIB")
    if not force and not is_stale():
        return LIB
    OBJ.mkdir(parents=True, exist_ok=True)
    jobs = [(CSRC / "mfcg_b200.cu", OBJ / "mfcg_b200.o", [])]
    jobs += [(CSRC / "mfcg_inst.cu", OBJ / f"mfcg_inst_p{p}.o", [f"-DMFCG_P={p}"]) for p in DEGREES]
    workers = min(len(jobs), os.cpu_count() or 4)
    with ThreadPoolExecutor(max_workers=workers) as pool:
        objs = list(pool.map(_compile, jobs))
    cmd = [_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(LIB), *map(str, objs)]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python -m paper_2205_08909_b200.build --variant tools/varlibs/x.so -DMFCG_TIMING ...
        i = sys.argv.index("--variant")
        flags = [a for a in sys.argv[i + 2:] if not a.startswith("--degrees=")]
        degs = [a for a in sys.argv[i + 2:] if a.startswith("--degrees=")]
        degrees = tuple(int(x) for x in degs[0].split("=")[1].split(",")) if degs else DEGREES
        build_variant(Path(sys.argv[i + 1]), flags, degrees=degrees, verbose=True)
    else:
        build_library(force="--force" in sys.argv, verbose=True)
