"""Structured hexahedral brick meshes and per-quadrature-point geometry (host side).

Mirrors the public surface of the reference's ``mfcg.mesh``
(``pkg/src/mfcg/mesh.py:26-37``): ``HexMesh``, ``GeometryVariant``,
``GeometryData``, ``build_cartesian_mesh``, ``deform_mesh``,
``quadratic_geometry_nodes``, ``geometry_data``, ``precompute_geometry``,
``compute_jacobians_from_nodes``, ``mesh_to_text`` / ``mesh_from_text``.

As in the reference (mesh.py:1-9) the authoritative cell map is the
tri-quadratic interpolant of ``x -> x + a * prod_d sin(pi x_d / L_d)`` through
the 3x3x3 lattice {0, 1/2, 1}^3 of every cell; all geometry variants describe
that same map.

Everything here is NumPy and exists for setup and for *checking* the GPU: the
device computes its own geometry tables (kernel ``k_geometry`` in
``csrc/mfcg_kernels.cuh``) from (cells, extents, deformation) because the
stored variants reach 9-15 GB at the benchmark sizes.  The host version
evaluates the tri-quadratic map by an explicit 27-term tensor table (not by
the reference's sweeps) and processes cells in chunks to bound memory.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from .tensor import QuadratureRule1D, gauss_lobatto_quadrature

__all__ = [
    "HexMesh",
    "GeometryVariant",
    "GeometryData",
    "build_cartesian_mesh",
    "deform_mesh",
    "quadratic_geometry_nodes",
    "geometry_data",
    "precompute_geometry",
    "compute_jacobians_from_nodes",
    "mesh_to_text",
    "mesh_from_text",
]

_CHUNK_CELLS = 8192


class GeometryVariant(Enum):
    """How the operator obtains J^-1 and w_q det J (reference mesh.py:40-47)."""

    AFFINE = "affine"
    QUADRATIC_COMPUTE = "quadratic_compute"
    ISOPARAMETRIC_COMPUTE = "isoparametric_compute"
    INVERSE_JACOBIAN_LOAD = "inverse_jacobian_load"
    FINAL_TENSOR_LOAD = "final_tensor_load"


@dataclass(frozen=True)
class HexMesh:
    """Axis-aligned structured mesh of [0,extents], optionally pushed through
    the boundary-preserving sine bump (reference mesh.py:50-80)."""

    cells_per_dim: tuple
    extents: tuple
    deformation: float = 0.0
    vertex_coordinates: np.ndarray = field(repr=False, compare=False, default=None)
    cell_vertex_indices: np.ndarray = field(repr=False, compare=False, default=None)

    @property
    def n_cells(self) -> int:
        nx, ny, nz = self.cells_per_dim
        return nx * ny * nz

    def cell_coords(self, cell: int) -> tuple:
        nx, ny, _ = self.cells_per_dim
        if not 0 <= cell < self.n_cells:
            raise IndexError(f"cell index {cell} out of range")
        return cell % nx, (cell // nx) % ny, cell // (nx * ny)

    def map_points(self, points: np.ndarray) -> np.ndarray:
        """Deformation map on undeformed coordinates (..., 3): the same bump is
        added to all three coordinates (reference mesh.py:73-80)."""
        pts = np.asarray(points, dtype=np.float64)
        if self.deformation == 0.0:
            return pts.copy()
        s = np.sin(np.pi * pts / np.asarray(self.extents))
        bump = s[..., 0:1] * s[..., 1:2] * s[..., 2:3]
        return pts + self.deformation * bump


def build_cartesian_mesh(cells_per_dim, extents=(1.0, 1.0, 1.0)) -> HexMesh:
    """Uniform mesh of the brick [0,extents]; vertices x-fastest, 8 vertex ids
    per cell in (x fastest, z slowest) corner order (reference mesh.py:83-107)."""
    cells = tuple(int(c) for c in cells_per_dim)
    ext = tuple(float(e) for e in extents)
    if len(cells) != 3 or any(c < 1 for c in cells):
        raise ValueError("cells_per_dim entries must be >= 1")
    if len(ext) != 3 or any(e <= 0 for e in ext):
        raise ValueError("extents must be positive")
    nx, ny, nz = cells
    gx = np.linspace(0.0, ext[0], nx + 1)
    gy = np.linspace(0.0, ext[1], ny + 1)
    gz = np.linspace(0.0, ext[2], nz + 1)
    verts = np.empty(((nz + 1), (ny + 1), (nx + 1), 3))
    verts[..., 0] = gx[None, None, :]
    verts[..., 1] = gy[None, :, None]
    verts[..., 2] = gz[:, None, None]
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = (i + (nx + 1) * (j + (ny + 1) * k)).ravel()
    corner = np.array([dx + (nx + 1) * (dy + (ny + 1) * dz)
                       for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)])
    conn = (base[:, None] + corner[None, :]).astype(np.int64)
    return HexMesh(cells, ext, 0.0, verts.reshape(-1, 3), conn)


def _lattice(mesh: HexMesh, cells: np.ndarray, t: np.ndarray) -> np.ndarray:
    """Undeformed coordinates (len(cells), len(t)^3, 3) of the per-cell tensor
    lattice with 1D reference positions `t`, x fastest."""
    nx, ny, _ = mesh.cells_per_dim
    h = np.array([mesh.extents[d] / mesh.cells_per_dim[d] for d in range(3)])
    cells = np.asarray(cells, dtype=np.int64)
    cidx = np.stack([cells % nx, (cells // nx) % ny, cells // (nx * ny)], axis=1)
    origin = cidx * h
    m = len(t)
    loc = np.empty((m, m, m, 3))
    loc[..., 0] = t[None, None, :] * h[0]
    loc[..., 1] = t[None, :, None] * h[1]
    loc[..., 2] = t[:, None, None] * h[2]
    return origin[:, None, :] + loc.reshape(1, m ** 3, 3)


_HALF = np.array([0.0, 0.5, 1.0])


def _quadratic_nodes(mesh: HexMesh, cells) -> np.ndarray:
    return mesh.map_points(_lattice(mesh, cells, _HALF))


def quadratic_geometry_nodes(mesh: HexMesh, cell: int) -> np.ndarray:
    """The 27 tri-quadratic support points of one cell, (27, 3), x fastest
    (reference mesh.py:141-147)."""
    mesh.cell_coords(cell)
    return _quadratic_nodes(mesh, np.array([cell]))[0]


def _quad1d(t: np.ndarray):
    """Values and derivatives of the quadratic Lagrange polynomials on
    {0, 1/2, 1} at positions t: two (len(t), 3) tables."""
    t = np.asarray(t, dtype=np.float64)
    val = np.stack([2.0 * (t - 0.5) * (t - 1.0), -4.0 * t * (t - 1.0), 2.0 * t * (t - 0.5)], axis=1)
    der = np.stack([4.0 * t - 3.0, 4.0 - 8.0 * t, 4.0 * t - 1.0], axis=1)
    return val, der


def _gradient_tables(points_1d: np.ndarray) -> np.ndarray:
    """T[j, q, n] = d phi_n / d xi_j at tensor point q (x fastest) for the 27
    tri-quadratic shape functions n (x fastest)."""
    v, d = _quad1d(points_1d)
    tabs = []
    for j in range(3):
        fx = d if j == 0 else v
        fy = d if j == 1 else v
        fz = d if j == 2 else v
        # index order (qz, qy, qx, nz, ny, nx)
        tab = np.einsum("ka,jb,ic->kjiabc", fz, fy, fx)
        tabs.append(tab.reshape(len(points_1d) ** 3, 27))
    return np.stack(tabs)


def compute_jacobians_from_nodes(nodes: np.ndarray, geo_basis, nq: int = None):
    """Jacobians jac[c, q, i, j] = d x_i / d xi_j of tri-quadratic cell maps
    given node coordinates (n, 27, 3) at the tensor points of
    ``geo_basis.quadrature`` (a ``TensorBasis1D`` of degree 2) or, when
    `geo_basis` is a plain 1D point array, at those points.  Raises
    ``ValueError`` on a non-positive determinant (reference mesh.py:268-280)."""
    pts = geo_basis.quadrature.points if hasattr(geo_basis, "quadrature") else np.asarray(geo_basis)
    tab = _gradient_tables(pts)
    jac = np.einsum("cni,jqn->cqij", nodes, tab)
    det = np.linalg.det(jac)
    if det.size and np.min(det) <= 0.0:
        raise ValueError(f"degenerate cell: min det J = {np.min(det):.3e}")
    return jac, det


def _chunks(n):
    for lo in range(0, n, _CHUNK_CELLS):
        yield np.arange(lo, min(lo + _CHUNK_CELLS, n))


def deform_mesh(mesh: HexMesh, amplitude: float) -> HexMesh:
    """Add `amplitude` to the bump; reject amplitudes that make det J <= 0 on
    the 3-point Gauss-Lobatto rule of any cell (reference mesh.py:110-123)."""
    new = HexMesh(mesh.cells_per_dim, mesh.extents, mesh.deformation + amplitude,
                  mesh.vertex_coordinates, mesh.cell_vertex_indices)
    if amplitude != 0.0:
        pts = gauss_lobatto_quadrature(3).points
        try:
            for cells in _chunks(new.n_cells):
                compute_jacobians_from_nodes(_quadratic_nodes(new, cells), pts)
        except ValueError as err:
            raise ValueError(
                f"deformation amplitude {new.deformation} produces a "
                f"non-positive Jacobian ({err})") from None
    return new


@dataclass(frozen=True)
class GeometryData:
    """Per-cell geometric payload of one variant; `doubles_per_cell` is the
    data volume streamed per cell (reference mesh.py:177-191)."""

    variant: GeometryVariant
    quadrature: QuadratureRule1D
    payload: dict
    doubles_per_cell: int


def _tensor_weights(quad: QuadratureRule1D) -> np.ndarray:
    w = quad.weights
    return (w[:, None, None] * w[None, :, None] * w[None, None, :]).ravel()


def _symmetric_coefficient(inv: np.ndarray, jxw: np.ndarray) -> np.ndarray:
    """J^-1 (w det J) J^-T in 6-storage (xx, yy, zz, xy, xz, yz)
    (reference mesh.py:194-201)."""
    full = np.einsum("cqij,cqkj->cqik", inv, inv) * jxw[..., None, None]
    return np.stack([full[..., 0, 0], full[..., 1, 1], full[..., 2, 2],
                     full[..., 0, 1], full[..., 0, 2], full[..., 1, 2]], axis=-1)


def precompute_geometry(mesh: HexMesh, variant: GeometryVariant,
                        quad: QuadratureRule1D) -> GeometryData:
    """Geometry payload of one variant for all cells (reference mesh.py:209-252).
    Payload keys and shapes are the reference's."""
    nq = len(quad)
    weights = _tensor_weights(quad)
    if variant == GeometryVariant.AFFINE:
        if mesh.deformation != 0.0:
            raise ValueError("affine geometry requires an undeformed mesh")
        h = np.array([mesh.extents[d] / mesh.cells_per_dim[d] for d in range(3)])
        payload = {"inverse_jacobian": np.diag(1.0 / h), "det_j": float(np.prod(h)),
                   "weights": weights}
        return GeometryData(variant, quad, payload, 10)
    if variant == GeometryVariant.QUADRATIC_COMPUTE:
        nodes = np.concatenate([_quadratic_nodes(mesh, c) for c in _chunks(mesh.n_cells)])
        return GeometryData(variant, quad, {"nodes": nodes, "weights": weights}, 81)
    if variant == GeometryVariant.ISOPARAMETRIC_COMPUTE:
        raise ValueError("isoparametric_compute is outside the B200 hot-path scope "
                         "(SURVEY.md section 2 row 4); use quadratic_compute")
    if variant not in (GeometryVariant.INVERSE_JACOBIAN_LOAD, GeometryVariant.FINAL_TENSOR_LOAD):
        raise ValueError(f"unknown geometry variant {variant}")
    invs, jxws = [], []
    for cells in _chunks(mesh.n_cells):
        jac, det = compute_jacobians_from_nodes(_quadratic_nodes(mesh, cells), quad.points)
        invs.append(np.linalg.inv(jac))
        jxws.append(det * weights)
    inv = np.concatenate(invs)
    jxw = np.concatenate(jxws)
    if variant == GeometryVariant.INVERSE_JACOBIAN_LOAD:
        return GeometryData(variant, quad, {"inverse_jacobian": inv, "jxw": jxw}, 10 * nq ** 3)
    sym = _symmetric_coefficient(inv, jxw)
    return GeometryData(variant, quad, {"final_tensor": sym, "jxw": jxw}, 7 * nq ** 3)


def geometry_data(mesh: HexMesh, cell: int, variant: GeometryVariant,
                  quad: QuadratureRule1D) -> dict:
    """Per-cell view of a variant's payload (reference mesh.py:255-265)."""
    mesh.cell_coords(cell)
    data = precompute_geometry(mesh, variant, quad)
    if variant == GeometryVariant.AFFINE:
        return dict(data.payload)
    per_cell = ("nodes", "inverse_jacobian", "jxw", "final_tensor")
    return {k: (v[cell] if k in per_cell else v) for k, v in data.payload.items()}


def mesh_to_text(mesh: HexMesh) -> str:
    """Key-value text form (reference mesh.py:283-290)."""
    c, e = mesh.cells_per_dim, mesh.extents
    return (f"cells = {c[0]},{c[1]},{c[2]}\n"
            f"extents = {e[0]!r},{e[1]!r},{e[2]!r}\n"
            f"deformation = {mesh.deformation!r}\n")


def mesh_from_text(text: str) -> HexMesh:
    """Inverse of :func:`mesh_to_text` (reference mesh.py:293-307)."""
    kv = {}
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if line:
            key, _, val = line.partition("=")
            kv[key.strip()] = val.strip()
    mesh = build_cartesian_mesh([int(v) for v in kv["cells"].split(",")],
                                [float(v) for v in kv["extents"].split(",")])
    amp = float(kv.get("deformation", "0.0"))
    return deform_mesh(mesh, amp) if amp != 0.0 else mesh
