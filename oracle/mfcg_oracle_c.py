"""ctypes wrapper of oracle/mfcg_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import it."""
import ctypes as C
import os
import subprocess
import time
from pathlib import Path

import numpy as np

import mfcg_oracle as orc

HERE = Path(__file__).resolve().parent
LIB = HERE / "libmfcg_oracle.so"
_lib = None


class _Problem(C.Structure):
    _fields_ = [("p", C.c_int), ("nq", C.c_int), ("n_cells", C.c_int64), ("n_dofs", C.c_int64),
                ("idx", C.c_void_p), ("cmask", C.c_void_p), ("S", C.c_void_p), ("D", C.c_void_p),
                ("G", C.c_void_p), ("per_cell", C.c_int)]


def available(build=True):
    global _lib
    if _lib is not None:
        return True
    src = HERE / "mfcg_oracle.c"
    if build and (not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime):
        try:
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True, capture_output=True)
        except Exception:
            return False
    if not LIB.exists():
        return False
    _lib = C.CDLL(str(LIB))
    _lib.oracle_max_threads.restype = C.c_int
    _lib.oracle_set_threads.argtypes = [C.c_int]
    _lib.oracle_apply.argtypes = [C.POINTER(_Problem), C.c_void_p, C.c_void_p]
    _lib.oracle_combined_pcg.argtypes = [C.POINTER(_Problem), C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                         C.c_void_p, C.c_void_p]
    _lib.oracle_combined_pcg.restype = C.c_int
    return True


class CProblem:
    """Same inputs as mfcg_oracle.Problem; owns the flattened tables the C code reads."""

    def __init__(self, prob: orc.Problem):
        assert available()
        self.prob = prob
        self.idx = np.ascontiguousarray(prob.idx, dtype=np.int64)
        self.cmask = np.ascontiguousarray(prob.cmask, dtype=np.uint8)
        self.S = np.ascontiguousarray(prob.S)
        self.D = np.ascontiguousarray(prob.D)
        if prob.geometry == "affine":
            G = prob.G(None)[None]
            per_cell = 0
        else:
            G = np.concatenate([prob.G(np.arange(lo, min(lo + 4096, prob.n_cells)))
                                for lo in range(0, prob.n_cells, 4096)])
            per_cell = 1
        self.G = np.ascontiguousarray(np.stack([G[..., 0, 0], G[..., 1, 1], G[..., 2, 2], G[..., 0, 1],
                                                G[..., 0, 2], G[..., 1, 2]], axis=-1))
        self.c = _Problem(prob.p, prob.nq, prob.n_cells, prob.n_dofs, self.idx.ctypes.data,
                          self.cmask.ctypes.data, self.S.ctypes.data, self.D.ctypes.data,
                          self.G.ctypes.data, per_cell)

    def apply(self, src):
        src = np.ascontiguousarray(src, dtype=np.float64)
        dst = np.empty_like(src)
        _lib.oracle_apply(C.byref(self.c), src.ctypes.data, dst.ctypes.data)
        return dst

    def combined_pcg(self, b, minv, iters, tol=1e-8):
        b = np.ascontiguousarray(b, dtype=np.float64)
        minv = np.ascontiguousarray(minv, dtype=np.float64)
        x = np.empty_like(b)
        hist = np.zeros((iters, 4))
        k = _lib.oracle_combined_pcg(C.byref(self.c), b.ctypes.data, minv.ctypes.data, iters, tol,
                                     x.ctypes.data, hist.ctypes.data)
        if k < 0:
            raise orc.Breakdown(f"breakdown at iteration {-k}")
        return x, k, hist[:k]


def max_threads():
    return _lib.oracle_max_threads() if available() else 1


def time_combined_pcg(cells, p, nq, blocks, constrained, n_dofs, b, iters, threads=None):
    """(seconds, threads) of `iters` merged Jacobi-PCG iterations on the host."""
    if threads and available():
        _lib.oracle_set_threads(int(threads))
    prob = orc.Problem(tuple(cells), (1.0, 1.0, 1.0), 0.0, p, nq, blocks, constrained, n_dofs)
    cp = CProblem(prob)
    minv = orc.inverse_diagonal(prob)
    cp.apply(b)  # warm up the thread pool
    t0 = time.perf_counter()
    cp.combined_pcg(b, minv, iters)
    return time.perf_counter() - t0, max_threads()
