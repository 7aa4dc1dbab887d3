"""Matrix-free Laplace operator on the GPU behind the reference's operator
protocol (``pkg/src/mfcg/operator.py:44``): ``OperatorSpec``,
``DiagonalPreconditioner``, ``MatrixFreeOperator``.

``MatrixFreeOperator(spec, mesh, handler, plan)`` keeps the reference's
constructor, public fields and error behaviour (operator.py:130-155) but owns a
device-resident operator in ``libmfcg_b200.so``: ``apply`` and
``compute_diagonal`` are single C-ABI calls, and ``solvers.solve`` hands the
whole CG loop to the library.  The hot path has no CPU implementation here:
without the library or a GPU the constructor raises.

Scope: the Laplace operator on 1 or 3 components (the
scalar operator acts on every component, operator.py:256-281); the mass
equations are rejected with ``NotImplementedError``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .dofs import RANGE_SIZE, BatchPlan, DofHandler, compute_range_schedule
from .mesh import GeometryVariant, HexMesh, precompute_geometry
from .tensor import gauss_lobatto_quadrature, gauss_quadrature, lagrange_basis

__all__ = ["OperatorSpec", "DiagonalPreconditioner", "MatrixFreeOperator"]

EQUATIONS = ("mass", "laplace", "mass_plus_laplace")


@dataclass(frozen=True)
class OperatorSpec:
    """Field-for-field the reference's spec (operator.py:49-82)."""

    equation: str
    components: int
    degree: int
    n_q_1d: int
    geometry: GeometryVariant
    quadrature_kind: str = "gauss"
    scaling: float = 1.0

    def __post_init__(self):
        if self.equation not in EQUATIONS:
            raise ValueError(f"unknown equation {self.equation!r}")
        if self.components not in (1, 3):
            raise ValueError("components must be 1 or 3")
        if self.degree < 1:
            raise ValueError("degree must be >= 1")
        if self.n_q_1d < self.degree + 1:
            raise ValueError("n_q_1d must be at least p+1")
        if self.quadrature_kind not in ("gauss", "gauss_lobatto"):
            raise ValueError(f"unknown quadrature {self.quadrature_kind!r}")
        if self.quadrature_kind == "gauss_lobatto" and self.n_q_1d != self.degree + 1:
            raise ValueError("gauss_lobatto requires n_q_1d == p+1 (collocation)")

    @property
    def needs_values(self) -> bool:
        return self.equation in ("mass", "mass_plus_laplace")

    @property
    def needs_gradients(self) -> bool:
        return self.equation in ("laplace", "mass_plus_laplace")


@dataclass(frozen=True)
class DiagonalPreconditioner:
    """Inverse operator diagonal per scalar node (operator.py:85-99).  When it
    comes from ``MatrixFreeOperator.compute_diagonal`` it remembers its
    operator, so ``solve`` can use the copy already resident on the GPU."""

    inverse_diagonal: np.ndarray
    _owner: object = None

    def full_vector(self, components: int) -> np.ndarray:
        return np.repeat(self.inverse_diagonal, components)

    def apply(self, r: np.ndarray, components: int) -> np.ndarray:
        if components == 1:
            return self.inverse_diagonal * r
        return (r.reshape(-1, components) * self.inverse_diagonal[:, None]).ravel()


def _as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


class MatrixFreeOperator:
    """v = A u on the B200 (reference class: operator.py:127-376)."""

    def __init__(self, spec: OperatorSpec, mesh: HexMesh, handler: DofHandler,
                 plan: BatchPlan, *, device: int = 0, precision: str = "fp64",
                 brick=(0, 0, 0), slab_z0: int = 0, global_cells_z: int = None):
        if spec.components != handler.components:
            raise ValueError("spec/handler component mismatch")
        if spec.degree != handler.degree:
            raise ValueError("spec/handler degree mismatch")
        if tuple(mesh.cells_per_dim) != tuple(handler.cells_per_dim):
            raise ValueError("mesh/handler shape mismatch")
        if spec.equation != "laplace":
            raise NotImplementedError(
                "the B200 hot path covers the Laplace operator (SURVEY.md section 8); "
                "mass equations are out of scope")
        if precision not in ("fp64", "fp32"):
            raise ValueError("precision must be 'fp64' or 'fp32'")
        self.spec = spec
        self.mesh = mesh
        self.handler = handler
        self.plan = plan
        self.precision = precision
        self.device = device
        self.quadrature = (gauss_quadrature(spec.n_q_1d) if spec.quadrature_kind == "gauss"
                           else gauss_lobatto_quadrature(spec.n_q_1d))
        self.basis = lagrange_basis(spec.degree, self.quadrature)
        self.n_dofs = handler.n_dofs
        self.components = spec.components
        self._geometry = None
        self._schedule = None
        self._handle = None
        self._lib = _lib.load()
        self._ctx = _lib.context(device)

        gl = gauss_lobatto_quadrature(spec.degree + 1)
        gl_basis = lagrange_basis(spec.degree, gl)
        keep = [_as_f64(self.basis.shape_values), _as_f64(self.basis.shape_gradients),
                _as_f64(self.quadrature.points), _as_f64(self.quadrature.weights),
                _as_f64(gl.points), _as_f64(gl.weights), _as_f64(gl_basis.shape_gradients),
                np.ascontiguousarray(handler.cell_index_blocks, dtype=np.int32),
                np.ascontiguousarray(handler.constrained_dofs, dtype=np.int64)]
        d = _lib.OpDesc()
        d.degree, d.n_q_1d = spec.degree, spec.n_q_1d
        (d.shape_values, d.shape_gradients, d.quad_points, d.quad_weights,
         d.gl_points, d.gl_weights, d.gl_gradients) = (_ptr(a) for a in keep[:7])
        d.cells = (C.c_int32 * 3)(*mesh.cells_per_dim)
        d.extents = (C.c_double * 3)(*mesh.extents)
        d.deformation = float(mesh.deformation)
        d.cell_index_blocks = _ptr(keep[7], C.c_int32)
        d.n_dofs = handler.n_dofs
        d.constrained = _ptr(keep[8], C.c_int64)
        d.n_constrained = keep[8].size
        d.geometry = _lib.GEOMETRY_CODES[spec.geometry.value] if spec.geometry.value in _lib.GEOMETRY_CODES else -1
        if d.geometry < 0:
            raise NotImplementedError(f"geometry variant {spec.geometry.value} is outside the hot-path scope")
        d.precision = 0 if precision == "fp64" else 1
        d.brick = (C.c_int32 * 3)(*brick)
        # z-slab of a larger mesh (slabs.py): `mesh` is the slab, its extents those of the whole mesh
        d.components = spec.components
        d.slab_z0 = int(slab_z0)
        d.global_cells_z = int(global_cells_z) if global_cells_z else mesh.cells_per_dim[2]
        self.slab_z0, self.global_cells_z = d.slab_z0, d.global_cells_z
        handle = C.c_void_p()
        _lib.check(self._lib.mfcg_op_create(self._ctx, C.byref(d), C.byref(handle)))
        self._handle = handle

    def __del__(self):
        handle, self._handle = getattr(self, "_handle", None), None
        if handle:
            try:
                self._lib.mfcg_op_destroy(handle)
            except Exception:
                pass

    # -- lazily built host-side data the reference exposes as attributes ------

    @property
    def geometry(self):
        """Host copy of the variant's payload (mesh.precompute_geometry); the
        device builds its own tables, this is for inspection and tests."""
        if self._geometry is None:
            self._geometry = precompute_geometry(self.mesh, self.spec.geometry, self.quadrature)
        return self._geometry

    @property
    def schedule(self):
        """64-entry range schedule of the batch plan (dofs.py:395-423); data
        only -- the GPU schedules by bricks."""
        if self._schedule is None:
            self._schedule = compute_range_schedule(self.handler, self.plan)
        return self._schedule

    def info(self) -> dict:
        out = _lib.OpInfo()
        _lib.check(self._lib.mfcg_op_get_info(self._handle, C.byref(out)))
        return {"n_dofs": out.n_dofs, "n_interior": out.n_interior, "n_bricks": out.n_bricks,
                "brick": tuple(out.brick), "threads": out.threads, "smem_bytes": out.smem_bytes,
                "geometry_bytes": out.geometry_bytes}

    def device_geometry(self) -> dict:
        """The geometry table the device built for a stored variant, under the reference's
        payload keys (mesh.py:243-251): ``final_tensor`` (n_cells, n_q^3, 6) or
        ``inverse_jacobian`` (n_cells, n_q^3, 3, 3) + ``jxw`` (n_cells, n_q^3)."""
        kind = _lib.GEOMETRY_CODES[self.spec.geometry.value]
        nc, nq3 = self.mesh.n_cells, self.spec.n_q_1d ** 3
        if kind == 1:
            out = np.empty(nc * nq3 * 6)
            _lib.check(self._lib.mfcg_op_geometry(self._handle, 1, _ptr(out), out.size))
            return {"final_tensor": out.reshape(nc, nq3, 6)}
        if kind == 2:
            out = np.empty(nc * nq3 * 10)
            _lib.check(self._lib.mfcg_op_geometry(self._handle, 2, _ptr(out), out.size))
            return {"inverse_jacobian": out[:nc * nq3 * 9].reshape(nc, nq3, 3, 3),
                    "jxw": out[nc * nq3 * 9:].reshape(nc, nq3)}
        raise ValueError("the operator holds no stored geometry table")

    def device_permutation(self) -> np.ndarray:
        """perm[node] = index in the library's brick numbering (component c of
        that node lives at ``c * stride + perm[node]`` on the device)."""
        perm = np.empty(self.n_dofs // self.components, dtype=np.int32)
        _lib.check(self._lib.mfcg_op_device_permutation(self._handle, _ptr(perm, C.c_int32)))
        return perm

    # -- application ----------------------------------------------------------

    def apply(self, src: np.ndarray, out: np.ndarray = None, recorder=None,
              src_name: str = "src", dst_name: str = "dst") -> np.ndarray:
        """dst = A src (operator.py:285-292).  `recorder` must be None: access
        tracing is CPU instrumentation outside the hot path."""
        if recorder is not None:
            raise NotImplementedError("access recorders are not supported on the GPU operator")
        if len(src) != self.n_dofs or (out is not None and len(out) != self.n_dofs):
            raise ValueError("vector length does not match handler")
        s = _as_f64(src)
        if out is not None and out.dtype == np.float64 and out.flags.c_contiguous:
            dst = out
        else:
            dst = np.empty(self.n_dofs)
        _lib.check(self._lib.mfcg_op_apply(self._handle, s.ctypes.data, dst.ctypes.data, 0))
        if out is not None and dst is not out:
            out[:] = dst
            return out
        return dst

    def apply_device(self, src_ptr: int, dst_ptr: int) -> None:
        """dst = A src on fp64 device buffers (caller numbering) given as raw
        pointers, e.g. ``torch.Tensor.data_ptr()``; the caller synchronises its
        own stream first."""
        _lib.check(self._lib.mfcg_op_apply(self._handle, src_ptr, dst_ptr, 1))

    def apply_with_callbacks(self, src: np.ndarray, dst: np.ndarray, pre_fn=None, post_fn=None, *,
                             recorder=None, merge_ranges: bool = True, checked: bool = False,
                             src_name: str = "src", dst_name: str = "dst") -> None:
        """Reference entry point operator.py:294-370.  Python callbacks cannot
        run inside a CUDA kernel, so this uses the three-phase form the
        contract allows (all pre over ascending 64-entry ranges, dst = A src,
        all post; cf. ArrayOperator, solvers.py:97-109).  The fused path is
        reached through ``solvers.solve``."""
        if len(src) != self.n_dofs or len(dst) != self.n_dofs:
            raise ValueError("vector length does not match handler")
        if checked and recorder is None:
            raise ValueError("checked mode needs a recorder")
        if recorder is not None:
            raise NotImplementedError("access recorders are not supported on the GPU operator")
        n = self.n_dofs
        if pre_fn is not None:
            for lo in range(0, n, RANGE_SIZE):
                pre_fn(lo, min(lo + RANGE_SIZE, n))
        self.apply(src, out=dst)
        if post_fn is not None:
            for lo in range(0, n, RANGE_SIZE):
                post_fn(lo, min(lo + RANGE_SIZE, n))

    # -- diagonal ---------------------------------------------------------------

    def compute_diagonal(self) -> DiagonalPreconditioner:
        """1/diag of the GL-collocation operator, constrained entries 1
        (operator.py:380-418); ValueError when not positive definite."""
        out = np.empty(self.n_dofs // self.components)
        _lib.check(self._lib.mfcg_op_diagonal(self._handle, out.ctypes.data, 0))
        return DiagonalPreconditioner(out, self)

    # assembly oracles (operator.py:422-477) are test infrastructure of the
    # reference and are not re-implemented.
