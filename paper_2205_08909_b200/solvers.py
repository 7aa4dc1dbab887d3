"""CG drivers on the GPU behind the reference's solver entry points
(``pkg/src/mfcg/solvers.py:28-33``): ``solve``, ``solve_cg``, ``solve_pcg``,
``solve_combined_cg``, ``solve_combined_pcg``, ``SolverConfig``,
``SolveResult``, ``SolverBreakdown``.

The whole iteration loop runs inside ``mfcg_solve`` (one C-ABI call per solve):
scalars, breakdown/stagnation rules (solvers.py:172-177, 706-764) and the
history stay on the device.  ``pipelined`` and ``sstep`` are comparison
variants outside the hot path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .operator import DiagonalPreconditioner, MatrixFreeOperator

__all__ = ["SolverBreakdown", "SolverConfig", "SolveResult", "solve_cg", "solve_pcg",
           "solve_combined_cg", "solve_combined_pcg", "solve", "VARIANTS"]

VARIANTS = ("cg", "pcg", "combined_cg", "combined_pcg")


class SolverBreakdown(RuntimeError):
    """The Krylov recurrence lost positive definiteness (solvers.py:36-37)."""


@dataclass(frozen=True)
class SolverConfig:
    """Field-for-field the reference's config (solvers.py:40-56); `fused`
    selects the fused brick kernel (default) or the three-kernel
    pre / mat-vec / post form for the combined variants."""

    tolerance: float = 1e-8
    max_iterations: int = 500
    s: int = 4
    fixed_iterations: int = None
    force_x_updates: bool = False
    drift_check_every: int = 50
    fused: bool = True

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.s < 1:
            raise ValueError("s must be at least 1")


@dataclass
class SolveResult:
    x: np.ndarray
    iterations: int
    residual: float
    converged: bool
    variant: str
    history: list = field(default_factory=list)
    region_seconds: dict = field(default_factory=dict)
    matvecs: int = 0
    drift: tuple = ()
    device_stats: dict = field(default_factory=dict)


_BREAKDOWN_TEXT = {
    1: "{name} breakdown: p^T A p = {v:.3e} <= 0 at iteration {k}",
    2: "combined PCG: preconditioned product r^T M^-1 r = {v:.3e} <= 0 at iteration {k} "
       "(preconditioner not SPD)",
    3: "combined recurrence collapsed: beta = {v:.3e} <= 0 at iteration {k} before convergence",
}


def _run(variant: str, A, b, minv, cfg: SolverConfig, recorder, *, location=0, x_out=None,
         time_kernels=False, out=None):
    if recorder is not None:
        raise NotImplementedError("access recorders are not supported on the GPU solvers")
    if not isinstance(A, MatrixFreeOperator):
        raise TypeError("the GPU solvers need a paper_2205_08909_b200 MatrixFreeOperator")
    n = A.n_dofs
    prec = variant in ("pcg", "combined_pcg")
    args = _lib.SolveArgs()
    keep = []
    if location == 0:
        if len(b) != n:
            raise ValueError("right-hand side length does not match operator")
        bb = np.ascontiguousarray(b, dtype=np.float64)
        keep.append(bb)
        args.b = bb.ctypes.data
        if out is not None:
            if out.dtype != np.float64 or not out.flags.c_contiguous or len(out) != n:
                raise ValueError("out must be a contiguous float64 array of length n_dofs")
            x = out
        else:
            x = np.empty(n)
        args.x = x.ctypes.data
    else:
        args.b = int(b)
        args.x = int(x_out)
        x = None
    args.inv_diag = None
    if prec:
        if minv is None:
            raise ValueError(("combined PCG" if variant == "combined_pcg" else "pcg")
                             + " requires a preconditioner")
        if isinstance(minv, DiagonalPreconditioner) and minv._owner is A:
            pass  # the library uses the diagonal it already holds on the device
        elif location == 0:
            m = minv.inverse_diagonal if isinstance(minv, DiagonalPreconditioner) else minv
            m = np.ascontiguousarray(m, dtype=np.float64)
            if len(m) * A.components != n:
                raise ValueError("preconditioner length does not match operator")
            keep.append(m)
            args.inv_diag = m.ctypes.data
        else:
            args.inv_diag = int(minv)
    args.variant = _lib.VARIANT_CODES[variant]
    args.location = location
    args.tolerance = cfg.tolerance
    args.max_iterations = cfg.max_iterations
    args.fixed_iterations = -1 if cfg.fixed_iterations is None else int(cfg.fixed_iterations)
    args.force_x_updates = int(bool(cfg.force_x_updates))
    args.fused = int(bool(cfg.fused))
    args.time_kernels = int(bool(time_kernels))
    limit = cfg.fixed_iterations or cfg.max_iterations
    hist = np.zeros((limit, 4))
    args.history = hist.ctypes.data_as(C.POINTER(C.c_double))
    res = _lib.SolveResultC()
    try:
        _lib.check(A._lib.mfcg_solve(A._handle, C.byref(args), C.byref(res)))
    except _lib.BreakdownSignal:
        name = {"cg": "CG", "pcg": "PCG"}.get(variant, "combined CG")
        raise SolverBreakdown(_BREAKDOWN_TEXT[res.breakdown].format(
            name=name, v=res.breakdown_value, k=res.breakdown_iteration)) from None
    k = res.iterations
    history = [{"k": i + 1, "alpha": float(hist[i, 0]), "beta": float(hist[i, 1]),
                "gamma": float(hist[i, 2]), "residual": float(hist[i, 3])} for i in range(k)]
    seconds = res.solve_ms * 1e-3
    regions = {"iteration": seconds} if variant.startswith("combined") else {"solve": seconds}
    if time_kernels:
        regions["matvec"] = res.operator_ms * 1e-3
    stats = {"solve_ms": res.solve_ms, "operator_ms": res.operator_ms,
             "kernel_launches": res.kernel_launches, "operator_launches": res.operator_launches,
             "bnorm": res.bnorm}
    return SolveResult(x, k, float(res.residual), bool(res.converged), variant, history,
                       regions, res.matvecs, (), stats)


def solve_cg(A, b, config: SolverConfig = None, *, recorder=None) -> SolveResult:
    """Textbook CG (solvers.py:183-254)."""
    return _run("cg", A, b, None, config or SolverConfig(), recorder)


def solve_pcg(A, b, minv, config: SolverConfig = None, *, recorder=None) -> SolveResult:
    """Jacobi-PCG, region-by-region kernels (solvers.py:257-340)."""
    return _run("pcg", A, b, minv, config or SolverConfig(), recorder)


def solve_combined_cg(A, b, config: SolverConfig = None, *, recorder=None) -> SolveResult:
    """Merged CG (solvers.py:795-802)."""
    return _run("combined_cg", A, b, None, config or SolverConfig(), recorder)


def solve_combined_pcg(A, b, minv, config: SolverConfig = None, *, recorder=None) -> SolveResult:
    """Merged Jacobi-PCG (solvers.py:805-813)."""
    if minv is None:
        raise ValueError("combined PCG requires a preconditioner")
    return _run("combined_pcg", A, b, minv, config or SolverConfig(), recorder)


def solve(variant: str, A, b, *, minv=None, config: SolverConfig = None, recorder=None,
          out: np.ndarray = None, time_kernels: bool = False) -> SolveResult:
    """Dispatch by variant name (solvers.py:816-834).  Extensions: `out` receives
    the solution (e.g. a pinned buffer) instead of a fresh array; `time_kernels`
    adds per-launch CUDA-event timing of the operator kernel to the result."""
    if out is not None or time_kernels:
        if variant not in VARIANTS:
            raise ValueError(f"unknown solver variant {variant!r}")
        if variant in ("pcg", "combined_pcg") and minv is None:
            raise ValueError(f"{variant} requires a preconditioner")
        return _run(variant, A, b, minv, config or SolverConfig(), recorder, out=out,
                    time_kernels=time_kernels)
    if variant == "cg":
        return solve_cg(A, b, config, recorder=recorder)
    if variant == "pcg":
        if minv is None:
            raise ValueError("pcg requires a preconditioner")
        return solve_pcg(A, b, minv, config, recorder=recorder)
    if variant == "combined_cg":
        return solve_combined_cg(A, b, config, recorder=recorder)
    if variant == "combined_pcg":
        return solve_combined_pcg(A, b, minv, config, recorder=recorder)
    if variant in ("pipelined", "sstep"):
        raise NotImplementedError(f"{variant!r} is a comparison variant outside the B200 hot path")
    raise ValueError(f"unknown solver variant {variant!r}")


def solve_device(variant: str, A, b_ptr: int, x_ptr: int, *, minv=None, minv_ptr: int = None,
                 config: SolverConfig = None, time_kernels: bool = False) -> SolveResult:
    """Same solve with b and x (and optionally 1/diag) resident on the GPU as
    fp64 buffers in the caller's numbering (raw device pointers).  `minv` may be
    the operator's own DiagonalPreconditioner (uses the cached device copy)."""
    m = minv if minv is not None else minv_ptr
    return _run(variant, A, b_ptr, m, config or SolverConfig(), None, location=1, x_out=x_ptr,
                time_kernels=time_kernels)
