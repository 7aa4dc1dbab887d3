"""ctypes binding of ``libmfcg_b200.so`` (declarations: ``include/mfcg_b200.h``).

There is no CPU fallback: if the library is missing or no B200 is visible,
every call raises.  The library is built in-tree by
:func:`paper_2205_08909_b200.build.build_library` (``__graft_entry__.build``).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# MFCG_LIB: explicit path of a variant build (timing experiments, -DMFCG_BOUNDS); the production
# library is never overwritten by experiments
LIB_PATH = Path(os.environ.get("MFCG_LIB") or Path(__file__).resolve().parent / "libmfcg_b200.so")

OK, EINVAL, ENOMEM, ECUDA, EBREAKDOWN, EUNSUPPORTED = range(6)

GEOMETRY_CODES = {
    "affine": 0,
    "final_tensor_load": 1,
    "inverse_jacobian_load": 2,
    "quadratic_compute": 3,
}
VARIANT_CODES = {"cg": 0, "pcg": 1, "combined_cg": 2, "combined_pcg": 3}

_dp = C.POINTER(C.c_double)


class OpDesc(C.Structure):
    _fields_ = [
        ("degree", C.c_int32), ("n_q_1d", C.c_int32),
        ("shape_values", _dp), ("shape_gradients", _dp),
        ("quad_points", _dp), ("quad_weights", _dp),
        ("gl_points", _dp), ("gl_weights", _dp), ("gl_gradients", _dp),
        ("cells", C.c_int32 * 3), ("extents", C.c_double * 3), ("deformation", C.c_double),
        ("cell_index_blocks", C.POINTER(C.c_int32)), ("n_dofs", C.c_int64),
        ("constrained", C.POINTER(C.c_int64)), ("n_constrained", C.c_int64),
        ("geometry", C.c_int32), ("precision", C.c_int32), ("brick", C.c_int32 * 3),
        ("slab_z0", C.c_int32), ("global_cells_z", C.c_int32), ("components", C.c_int32),
    ]


class OpInfo(C.Structure):
    _fields_ = [
        ("n_dofs", C.c_int64), ("n_interior", C.c_int64), ("n_bricks", C.c_int64),
        ("brick", C.c_int32 * 3), ("threads", C.c_int32), ("smem_bytes", C.c_int32),
        ("geometry_bytes", C.c_int64),
    ]


class SolveArgs(C.Structure):
    _fields_ = [
        ("variant", C.c_int32), ("location", C.c_int32),
        ("b", C.c_void_p), ("inv_diag", C.c_void_p), ("x", C.c_void_p),
        ("tolerance", C.c_double), ("max_iterations", C.c_int32),
        ("fixed_iterations", C.c_int32), ("force_x_updates", C.c_int32),
        ("fused", C.c_int32), ("time_kernels", C.c_int32), ("history", _dp),
    ]


class SolveResultC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("converged", C.c_int32), ("matvecs", C.c_int32),
        ("breakdown", C.c_int32), ("breakdown_iteration", C.c_int32),
        ("breakdown_value", C.c_double), ("residual", C.c_double), ("bnorm", C.c_double),
        ("solve_ms", C.c_double), ("operator_ms", C.c_double),
        ("kernel_launches", C.c_int64), ("operator_launches", C.c_int64),
    ]


EXPORTS = (
    "mfcg_ctx_create", "mfcg_ctx_destroy", "mfcg_ctx_stream", "mfcg_last_error", "mfcg_op_create",
    "mfcg_op_destroy", "mfcg_op_get_info", "mfcg_op_device_permutation",
    "mfcg_op_apply", "mfcg_op_diagonal", "mfcg_op_geometry", "mfcg_solve",
    "mfcg_comm_unique_id", "mfcg_ctx_init_comm", "mfcg_apply_group", "mfcg_diagonal_group",
    "mfcg_solve_group",
)

_lib = None


def load():
    """Load the shared library (once) and declare the prototypes."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 hot path)")
    lib = C.CDLL(str(LIB_PATH))
    vp = C.c_void_p
    lib.mfcg_last_error.restype = C.c_char_p
    lib.mfcg_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    lib.mfcg_ctx_destroy.argtypes = [vp]
    lib.mfcg_ctx_stream.argtypes = [vp]
    lib.mfcg_ctx_stream.restype = vp
    lib.mfcg_ctx_destroy.restype = None
    lib.mfcg_op_create.argtypes = [vp, C.POINTER(OpDesc), C.POINTER(vp)]
    lib.mfcg_op_destroy.argtypes = [vp]
    lib.mfcg_op_destroy.restype = None
    lib.mfcg_op_get_info.argtypes = [vp, C.POINTER(OpInfo)]
    lib.mfcg_op_device_permutation.argtypes = [vp, C.POINTER(C.c_int32)]
    lib.mfcg_op_apply.argtypes = [vp, vp, vp, C.c_int]
    lib.mfcg_op_diagonal.argtypes = [vp, vp, C.c_int]
    lib.mfcg_op_geometry.argtypes = [vp, C.c_int, _dp, C.c_int64]
    lib.mfcg_solve.argtypes = [vp, C.POINTER(SolveArgs), C.POINTER(SolveResultC)]
    lib.mfcg_comm_unique_id.argtypes = [vp]
    lib.mfcg_ctx_init_comm.argtypes = [vp, vp, C.c_int, C.c_int]
    lib.mfcg_apply_group.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(vp), C.POINTER(vp), C.c_int]
    lib.mfcg_diagonal_group.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(vp), C.c_int]
    lib.mfcg_solve_group.argtypes = [C.POINTER(vp), C.c_int, C.POINTER(SolveArgs), C.POINTER(SolveResultC)]
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().mfcg_last_error()
    return msg.decode() if msg else ""


class BreakdownSignal(RuntimeError):
    """Raised by :func:`check` for MFCG_EBREAKDOWN; solvers.py turns it into
    ``SolverBreakdown`` with the reference's wording."""


def check(status: int):
    if status == OK:
        return
    msg = last_error()
    if status == EINVAL:
        raise ValueError(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    if status == EBREAKDOWN:
        raise BreakdownSignal(msg)
    if status == EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


_contexts = {}


def context(device: int = 0):
    """One library context (CUDA stream) per device, created on first use."""
    if device not in _contexts:
        lib = load()
        ctx = C.c_void_p()
        check(lib.mfcg_ctx_create(device, C.byref(ctx)))
        _contexts[device] = ctx
    return _contexts[device]


def stream_handle(device: int = 0) -> int:
    """Raw cudaStream_t of the library context (wrap with torch.cuda.ExternalStream)."""
    return int(load().mfcg_ctx_stream(context(device)))
