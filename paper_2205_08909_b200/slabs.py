"""z-slab decomposition of the structured mesh across GPUs (BASELINE configs[4]).

The reference is single-process; the paper's scheme is realised as:
rank g owns the cell layers ``[z0, z0 + nz_g)``; two adjacent slabs share exactly one lattice
plane of ``(nx p + 1)(ny p + 1)`` DoFs, held by both (the lower slab owns it for the dot
products, the upper one flags it as a ghost copy).  Per merged iteration each slab adds the
neighbour's partial ``v`` on that plane (one plane each way, overlapped with the interior brick
layers) and the seven sums go through one all-reduce.  ``r, p, x`` on the plane are updated
redundantly on both sides from identical inputs, so no second exchange is needed.

Host-side tables come from the package's own ``distribute_dofs`` on the slab mesh; the
constraint set and the local->global map are derived from the global lattice.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib, dofs
from .dofs import DofHandler
from .mesh import HexMesh, build_cartesian_mesh

__all__ = ["slab_layers", "Slab", "build_slab", "renumber_slab", "interface_plane_nodes", "SlabGroup"]


def slab_layers(nz: int, n_slabs: int):
    """[(z0, nz_g)]: cell layers of every slab, as even as possible, lower slabs first."""
    if n_slabs < 1 or n_slabs > nz:
        raise ValueError("need 1 <= n_slabs <= cell layers")
    base, extra = divmod(nz, n_slabs)
    out, z0 = [], 0
    for g in range(n_slabs):
        n = base + (1 if g < extra else 0)
        out.append((z0, n))
        z0 += n
    return out


@dataclass(frozen=True)
class Slab:
    mesh: HexMesh            # cells of the slab, extents/deformation of the whole mesh
    handler: DofHandler      # default numbering of the slab lattice, global Dirichlet set restricted
    z0: int
    global_cells_z: int
    global_nodes: np.ndarray  # local node -> lattice id I + NX (J + NY K_global) of the whole mesh

    @property
    def has_lower(self):
        return self.z0 > 0

    @property
    def has_upper(self):
        return self.z0 + self.mesh.cells_per_dim[2] < self.global_cells_z


def _lattice_ids(handler: DofHandler, z0: int):
    """(local node ids, I, J, K_global) for every (cell, local node), flattened."""
    p = handler.degree
    nx, ny, nz = handler.cells_per_dim
    n1 = p + 1
    cells = np.arange(handler.n_cells)
    idx = dofs.expand_batch(handler, cells)                       # (n_cells, n1^3)
    cx, cy, cz = cells % nx, (cells // nx) % ny, cells // (nx * ny)
    k, j, i = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    I = (cx[:, None] * p + i.ravel()[None, :]).ravel()
    J = (cy[:, None] * p + j.ravel()[None, :]).ravel()
    K = (cz[:, None] * p + k.ravel()[None, :]).ravel() + z0 * p
    return idx.ravel(), I, J, K


def build_slab(global_mesh: HexMesh, p: int, z0: int, nz_g: int, constrain_boundary: bool = True,
               components: int = 1) -> Slab:
    """Tables of one slab: the slab mesh, its handler with the global Dirichlet set restricted to
    the slab (interface planes are NOT constrained), and the local->global lattice map (per node;
    with 3 components unknown ``3 * node + c`` of the slab is unknown ``3 * global_node + c`` of the mesh)."""
    nx, ny, nz = global_mesh.cells_per_dim
    mesh = replace(build_cartesian_mesh((nx, ny, nz_g), global_mesh.extents),
                   extents=global_mesh.extents, deformation=global_mesh.deformation)
    hs = dofs.distribute_dofs(mesh, p, 1, constrain_boundary=False)
    node, I, J, K = _lattice_ids(hs, z0)
    NX, NY, NZ = nx * p + 1, ny * p + 1, nz * p + 1
    glob = np.empty(hs.n_dofs, dtype=np.int64)
    glob[node] = I + NX * (J + NY * K)
    constrained = np.empty(0, dtype=np.int64)
    if constrain_boundary:
        on = (I == 0) | (I == NX - 1) | (J == 0) | (J == NY - 1) | (K == 0) | (K == NZ - 1)
        constrained = np.unique(node[on])
    h = hs if components == 1 else dofs.distribute_dofs(mesh, p, components, constrain_boundary=False)
    if components > 1:  # constraints cover whole nodes (dofs.py:174-178)
        constrained = (constrained[:, None] * components + np.arange(components)[None, :]).ravel()
    h = DofHandler(h.n_dofs, components, p, mesh.cells_per_dim, h.cell_index_blocks, constrained)
    return Slab(mesh, h, z0, nz, glob)


def renumber_slab(slab: Slab, plan) -> Slab:
    """`renumber_optimized` on a slab with its interface planes in the remote-shared category (
    the reference's placeholder dofs.py:307-310): unknowns touched by one batch first, then those shared between
    batches, then the planes shared with the neighbouring slabs (contiguous: PAPER.md:6247-6253), the Dirichlet
    unknowns last.  `global_nodes` follows the permutation."""
    remote = []
    if slab.has_lower:
        remote.append(interface_plane_nodes(slab, "lower"))
    if slab.has_upper:
        remote.append(interface_plane_nodes(slab, "upper"))
    remote = np.concatenate(remote) if remote else np.empty(0, dtype=np.int64)
    h = dofs.renumber_optimized(slab.handler, plan, remote_shared=remote)
    glob = np.empty_like(slab.global_nodes)
    glob[h.permutation] = slab.global_nodes
    return Slab(slab.mesh, h, slab.z0, slab.global_cells_z, glob)


def interface_plane_nodes(slab: Slab, side: str) -> np.ndarray:
    """Local node ids of the slab's bottom ('lower') or top ('upper') lattice plane, ordered by
    global lattice id -- the ghost map of that interface."""
    p = slab.handler.degree
    nx, ny, _ = slab.mesh.cells_per_dim
    NX, NY = nx * p + 1, ny * p + 1
    Kg = slab.global_nodes // (NX * NY)
    K = slab.z0 * p if side == "lower" else (slab.z0 + slab.mesh.cells_per_dim[2]) * p
    nodes = np.flatnonzero(Kg == K)
    return nodes[np.argsort(slab.global_nodes[nodes], kind="stable")]


class SlabGroup:
    """Adjacent slabs held by this process (bottom to top) driven in lockstep through
    ``mfcg_apply_group / mfcg_diagonal_group / mfcg_solve_group``.  With one process per GPU the
    group has one member and the neighbours are NCCL ranks (``init_comm`` first)."""

    def __init__(self, ops):
        self.ops = list(ops)
        self._lib = _lib.load()
        self._handles = (C.c_void_p * len(self.ops))(*[op._handle for op in self.ops])

    def _ptr_array(self, arrays):
        return (C.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])

    def apply(self, srcs):
        srcs = [np.ascontiguousarray(s, dtype=np.float64) for s in srcs]
        dsts = [np.empty_like(s) for s in srcs]
        _lib.check(self._lib.mfcg_apply_group(self._handles, len(self.ops), self._ptr_array(srcs),
                                              self._ptr_array(dsts), 0))
        return dsts

    def compute_diagonal(self):
        outs = [np.empty(op.n_dofs // op.components) for op in self.ops]   # one value per node (operator.py:90)
        _lib.check(self._lib.mfcg_diagonal_group(self._handles, len(self.ops), self._ptr_array(outs), 0))
        return outs

    def solve(self, variant, bs, config=None, *, location=0, xs=None, minvs=None, outs=None):
        """(P)CG on the whole mesh, merged (`combined_cg`, `combined_pcg`) or standard (`cg`, `pcg`); returns one
        SolveResult per slab (same history).  ``minvs``: one caller-supplied inverse diagonal per slab (host arrays,
        one value per node) instead of the operator's own Jacobi diagonal.  Operators with 3 components (BP4 type)
        take interleaved vectors, as everywhere in the package."""
        from .solvers import SolveResult, SolverBreakdown, SolverConfig, _BREAKDOWN_TEXT
        cfg = config or SolverConfig()
        n = len(self.ops)
        limit = cfg.fixed_iterations or cfg.max_iterations
        args = (_lib.SolveArgs * n)()
        res = (_lib.SolveResultC * n)()
        keep, hists, xouts = [], [], []
        for g, op in enumerate(self.ops):
            a = args[g]
            if location == 0:
                b = np.ascontiguousarray(bs[g], dtype=np.float64)
                if len(b) != op.n_dofs:
                    raise ValueError("right-hand side length does not match operator")
                x = outs[g] if outs is not None else np.empty(op.n_dofs)   # `outs`: e.g. pinned host arrays
                if len(x) != op.n_dofs or x.dtype != np.float64 or not x.flags.c_contiguous:
                    raise ValueError("output array must be contiguous float64 of the operator's length")
                keep.append(b)
                a.b, a.x = b.ctypes.data, x.ctypes.data
                xouts.append(x)
            else:
                a.b, a.x = int(bs[g]), int(xs[g])
                xouts.append(None)
            a.inv_diag = None
            if minvs is not None:
                if location != 0:
                    raise ValueError("caller-supplied preconditioners are host arrays (location=0)")
                md = np.ascontiguousarray(getattr(minvs[g], "inverse_diagonal", minvs[g]), dtype=np.float64)
                if len(md) != op.n_dofs // op.components:   # one value per node (solvers.py:617-621)
                    raise ValueError("preconditioner length does not match operator")
                keep.append(md)
                a.inv_diag = md.ctypes.data
            a.variant = _lib.VARIANT_CODES[variant]
            a.location = location
            a.tolerance = cfg.tolerance
            a.max_iterations = cfg.max_iterations
            a.fixed_iterations = -1 if cfg.fixed_iterations is None else int(cfg.fixed_iterations)
            a.force_x_updates = int(bool(cfg.force_x_updates))
            a.fused = 1
            hist = np.zeros((limit, 4))
            hists.append(hist)
            a.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        try:
            _lib.check(self._lib.mfcg_solve_group(self._handles, n, args, res))
        except _lib.BreakdownSignal:
            r0 = res[0]
            raise SolverBreakdown(_BREAKDOWN_TEXT[r0.breakdown].format(
                name="combined CG", v=r0.breakdown_value, k=r0.breakdown_iteration)) from None
        out = []
        for g in range(n):
            k = res[g].iterations
            history = [{"k": i + 1, "alpha": float(hists[g][i, 0]), "beta": float(hists[g][i, 1]),
                        "gamma": float(hists[g][i, 2]), "residual": float(hists[g][i, 3])} for i in range(k)]
            out.append(SolveResult(xouts[g], k, float(res[g].residual), bool(res[g].converged), variant, history,
                                   {"iteration": res[g].solve_ms * 1e-3}, res[g].matvecs, (),
                                   {"solve_ms": res[g].solve_ms, "kernel_launches": res[g].kernel_launches,
                                    "operator_launches": res[g].operator_launches, "bnorm": res[g].bnorm}))
        return out


def init_comm(device: int, unique_id: bytes, rank: int, n_ranks: int) -> None:
    """Attach the NCCL communicator of a one-slab-per-process run to the device's context."""
    lib = _lib.load()
    buf = C.create_string_buffer(unique_id, 128)
    _lib.check(lib.mfcg_ctx_init_comm(_lib.context(device), buf, rank, n_ranks))


def new_unique_id() -> bytes:
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    _lib.check(lib.mfcg_comm_unique_id(buf))
    return buf.raw
