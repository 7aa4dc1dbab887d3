"""DoF numbering, cell batches, locality renumbering and the 64-entry range
schedule -- vectorised host code, bit-exact against the reference.

Public surface = the reference's ``mfcg.dofs`` (``pkg/src/mfcg/dofs.py:21-33``):
``DofHandler``, ``BatchPlan``, ``RangeSchedule``, ``RANGE_SIZE``,
``distribute_dofs``, ``batch_size``, ``make_batches``, ``renumber_optimized``,
``compute_range_schedule``, ``expand_cell_indices``, ``expand_batch``.

The reference builds these tables with Python loops and dictionaries
(dofs.py:138-179, 286-388); at the benchmark sizes (4e6 cells) that takes
minutes to hours, so every table here is derived in closed form on the
refined (2n+1)^3 entity lattice with NumPy sorts.  The *results* are required
to be identical integer for integer (tests/test_dofs_parity.py, golden
fixtures generated from the reference by oracle/make_golden.py).

The B200-specific "brick" numbering used inside the GPU library is not part of
this module's reference surface; its NumPy mirror lives in
:mod:`paper_2205_08909_b200.bricks`.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .mesh import HexMesh

__all__ = [
    "DofHandler",
    "BatchPlan",
    "RangeSchedule",
    "RANGE_SIZE",
    "distribute_dofs",
    "batch_size",
    "make_batches",
    "renumber_optimized",
    "compute_range_schedule",
    "expand_cell_indices",
    "expand_batch",
]

RANGE_SIZE = 64


@dataclass(frozen=True)
class DofHandler:
    """Numbering of a continuous Lagrange space on a structured hex mesh
    (field-for-field the reference's, dofs.py:38-62)."""

    n_dofs: int
    components: int
    degree: int
    cells_per_dim: tuple
    cell_index_blocks: np.ndarray = field(repr=False, compare=False)
    constrained_dofs: np.ndarray = field(repr=False, compare=False)
    numbering_kind: str = "default-cell-order"
    permutation: np.ndarray = field(repr=False, compare=False, default=None)

    @property
    def n_cells(self) -> int:
        nx, ny, nz = self.cells_per_dim
        return nx * ny * nz

    @property
    def n_nodes(self) -> int:
        return self.n_dofs // self.components

    @property
    def dofs_per_cell(self) -> int:
        return (self.degree + 1) ** 3 * self.components


@dataclass(frozen=True)
class BatchPlan:
    """Cells grouped into batches (reference dofs.py:65-75)."""

    batch_size: int
    batches: tuple
    traversal: str

    @property
    def n_batches(self) -> int:
        return len(self.batches)


@dataclass(frozen=True)
class RangeSchedule:
    """First/last touching batch per 64-entry range and the per-batch pre/post
    lists (reference dofs.py:78-96)."""

    range_size: int
    n_dofs: int
    first_touch_batch: np.ndarray = field(repr=False, compare=False)
    last_touch_batch: np.ndarray = field(repr=False, compare=False)
    pre_schedule: tuple = field(repr=False, compare=False)
    post_schedule: tuple = field(repr=False, compare=False)

    @property
    def n_ranges(self) -> int:
        return len(self.first_touch_batch)

    def range_bounds(self, r: int) -> tuple:
        lo = r * self.range_size
        return lo, min(lo + self.range_size, self.n_dofs)


# ---------------------------------------------------------------------------
# entity bookkeeping on the refined lattice
#
# Per direction a local node sits in slot 0 (low face), 1 (interior) or 2 (high
# face); an entity of a cell is a slot triple, stored at column sx+3sy+9sz of
# the block table (reference dofs.py:99-116).  Globally an entity is a point
# of the (2n+1)^3 "refined" lattice with coordinate 2*cell+slot.


def _slot_extent(p: int, slot):
    return np.where(np.asarray(slot) == 1, p - 1, 1)


@lru_cache(maxsize=None)
def _local_template(p: int):
    """(column, offset) per local node, x fastest: index = blocks[cell, column]
    + offset (reference dofs.py:119-135)."""
    n = p + 1
    a = np.arange(n)
    slot = np.where(a == 0, 0, np.where(a == p, 2, 1))
    inner = np.where(slot == 1, a - 1, 0)
    ext = _slot_extent(p, slot)
    col = (slot[None, None, :] + 3 * slot[None, :, None] + 9 * slot[:, None, None])
    off = inner[None, None, :] + ext[None, None, :] * (
        inner[None, :, None] + ext[None, :, None] * inner[:, None, None])
    col = np.broadcast_to(col, (n, n, n)).ravel().copy()
    off = np.broadcast_to(off, (n, n, n)).ravel().astype(np.int64)
    col.setflags(write=False)
    off.setflags(write=False)
    return col, off


def _axis_owner(n_cells_1d: int):
    """For every refined coordinate R in [0, 2n]: the first cell (lowest index)
    touching it and the slot that cell sees it in."""
    R = np.arange(2 * n_cells_1d + 1)
    owner = np.where(R % 2 == 1, (R - 1) // 2, np.maximum(R // 2 - 1, 0))
    return owner, R - 2 * owner


def distribute_dofs(mesh: HexMesh, p: int, components: int = 1,
                    constrain_boundary: bool = False) -> DofHandler:
    """Entity-block numbering: cells in lexicographic order, the 27 entities
    of a cell walked sx fastest, every entity seen for the first time gets the
    next contiguous block (reference dofs.py:138-179).

    Closed form: the first cell to see refined point (Rx,Ry,Rz) is the
    per-direction lowest touching cell, so sorting all entities by
    (owner cell, column in that cell) and prefix-summing their sizes
    reproduces the walk."""
    if p < 1:
        raise ValueError("degree must be >= 1")
    if components not in (1, 3):
        raise ValueError("components must be 1 or 3")
    nx, ny, nz = mesh.cells_per_dim
    own, slot, ext = [], [], []
    for n in (nx, ny, nz):
        o, s = _axis_owner(n)
        own.append(o)
        slot.append(s)
        ext.append(_slot_extent(p, np.arange(2 * n + 1) % 2))
    # refined lattice arrays indexed [Rz, Ry, Rx]
    size = (ext[2][:, None, None] * ext[1][None, :, None] * ext[0][None, None, :]).astype(np.int64)
    owner_cell = (own[0][None, None, :] + nx * (own[1][None, :, None] + ny * own[2][:, None, None]))
    column = slot[0][None, None, :] + 3 * slot[1][None, :, None] + 9 * slot[2][:, None, None]
    key = (owner_cell.astype(np.int64) * 27 + column).ravel()
    order = np.argsort(key, kind="stable")
    sizes_sorted = size.ravel()[order]
    starts_sorted = np.cumsum(sizes_sorted) - sizes_sorted
    start = np.empty(key.size, dtype=np.int64)
    start[order] = starts_sorted
    n_nodes = int(sizes_sorted.sum())
    start = np.where(size.ravel() == 0, -1, start).reshape(size.shape)

    cz, cy, cx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    blocks = np.empty((nx * ny * nz, 27), dtype=np.int32)
    for sz in range(3):
        for sy in range(3):
            for sx in range(3):
                blocks[:, sx + 3 * sy + 9 * sz] = start[2 * cz + sz, 2 * cy + sy, 2 * cx + sx].ravel()

    n_dofs = n_nodes * components
    constrained = np.empty(0, dtype=np.int64)
    if constrain_boundary:
        Rz, Ry, Rx = np.meshgrid(np.arange(2 * nz + 1), np.arange(2 * ny + 1),
                                 np.arange(2 * nx + 1), indexing="ij")
        on_bnd = ((Rx == 0) | (Rx == 2 * nx) | (Ry == 0) | (Ry == 2 * ny)
                  | (Rz == 0) | (Rz == 2 * nz)) & (size > 0)
        s0 = start[on_bnd]
        sz_ = size[on_bnd]
        nodes = np.repeat(s0, sz_) + _ragged_arange(sz_)
        nodes = np.sort(nodes)
        constrained = (nodes[:, None] * components + np.arange(components)).ravel()
    return DofHandler(n_dofs, components, p, mesh.cells_per_dim, blocks,
                      constrained.astype(np.int64))


def _ragged_arange(lengths: np.ndarray) -> np.ndarray:
    """Concatenation of arange(l) for l in lengths."""
    lengths = np.asarray(lengths, dtype=np.int64)
    total = int(lengths.sum())
    if total == 0:
        return np.empty(0, dtype=np.int64)
    ends = np.cumsum(lengths)
    return np.arange(total, dtype=np.int64) - np.repeat(ends - lengths, lengths)


def _expand_scalar(handler: DofHandler, cells: np.ndarray) -> np.ndarray:
    col, off = _local_template(handler.degree)
    return handler.cell_index_blocks[np.asarray(cells)][:, col].astype(np.int64) + off


def expand_batch(handler: DofHandler, cells) -> np.ndarray:
    """(len(cells), dofs_per_cell) global indices, nodes x fastest, components
    interleaved per node (reference dofs.py:229-236)."""
    scalar = _expand_scalar(handler, np.asarray(cells))
    c = handler.components
    if c == 1:
        return scalar
    return (scalar[..., None] * c + np.arange(c)).reshape(scalar.shape[0], -1)


def expand_cell_indices(handler: DofHandler, cell: int) -> np.ndarray:
    """Global indices of one cell (reference dofs.py:221-226)."""
    if not 0 <= cell < handler.n_cells:
        raise IndexError(f"cell index {cell} out of range")
    return expand_batch(handler, np.array([cell]))[0]


# ---------------------------------------------------------------------------
# batching


def batch_size(p: int, components: int, simd_lanes: int) -> int:
    """Cells per batch (reference dofs.py:243-248): about 1024 temporaries per
    lane, at least 2, times the lane count."""
    if p < 1 or components < 1 or simd_lanes < 1:
        raise ValueError("all batch-size inputs must be >= 1")
    per_lane = 1024 // (components * (p + 1) ** 3)
    return (per_lane if per_lane > 2 else 2) * simd_lanes


def _spread3(v: np.ndarray, bits: int) -> np.ndarray:
    out = np.zeros_like(v)
    for b in range(bits):
        out |= ((v >> b) & 1) << (3 * b)
    return out


def _morton_order(cells_per_dim) -> np.ndarray:
    """Cells sorted by Morton code, x bits lowest (reference dofs.py:251-264)."""
    nx, ny, nz = cells_per_dim
    bits = max(int(max(n - 1, 0)).bit_length() for n in cells_per_dim)
    cz, cy, cx = np.meshgrid(np.arange(nz, dtype=np.int64), np.arange(ny, dtype=np.int64),
                             np.arange(nx, dtype=np.int64), indexing="ij")
    code = (_spread3(cx, bits) | (_spread3(cy, bits) << 1) | (_spread3(cz, bits) << 2)).ravel()
    return np.argsort(code, kind="stable").astype(np.int64)


def make_batches(mesh: HexMesh, size: int, traversal: str = "lexicographic") -> BatchPlan:
    """Order cells by traversal, chunk into batches (reference dofs.py:267-279)."""
    if size < 1:
        raise ValueError("batch size must be >= 1")
    if traversal == "lexicographic":
        order = np.arange(mesh.n_cells, dtype=np.int64)
    elif traversal == "morton":
        order = _morton_order(mesh.cells_per_dim)
    else:
        raise ValueError(f"unknown traversal {traversal!r}")
    return BatchPlan(size, tuple(order[i:i + size] for i in range(0, len(order), size)), traversal)


def _cell_batch_ids(plan: BatchPlan, n_cells: int) -> np.ndarray:
    out = np.empty(n_cells, dtype=np.int64)
    lens = np.fromiter((len(c) for c in plan.batches), dtype=np.int64, count=plan.n_batches)
    out[np.concatenate(plan.batches) if plan.n_batches else np.empty(0, np.int64)] = \
        np.repeat(np.arange(plan.n_batches), lens)
    return out


# ---------------------------------------------------------------------------
# renumbering


def renumber_optimized(handler: DofHandler, plan: BatchPlan, remote_shared=None) -> DofHandler:
    """Locality renumbering of the batched cell loop (reference dofs.py:304-375).

    ``remote_shared`` (scalar node ids, default none): nodes shared with other processes.  The reference keeps
    category 2 for them "structurally present, always empty in this single-process build" (dofs.py:307-310,
    331, 354); the z-slab decomposition fills it with the interface planes, ordered like
    the reference orders that category: by (first batch, last batch, old start).  Without it the result is
    the reference's, bit for bit.

    Entity categories: (0) touched by exactly one batch, ordered by
    (batch, old start); (1) touched by several batches, ordered by
    (-(first+last), last-first, old start); (2) remote-shared, always empty in
    a single-process build; (3) constrained, ordered by (first, last, old
    start) at the very end.  Entity blocks stay contiguous.  Returns a new
    handler with ``permutation[old] = new``."""
    if handler.numbering_kind != "default-cell-order":
        raise ValueError("handler already renumbered")
    comp = handler.components
    p = handler.degree
    blocks = handler.cell_index_blocks
    n_nodes = handler.n_nodes

    col_size = np.array([int(np.prod(_slot_extent(p, [e % 3, (e // 3) % 3, e // 9])))
                         for e in range(27)], dtype=np.int64)
    flat = blocks.ravel().astype(np.int64)
    valid = flat >= 0
    cell_of = np.repeat(np.arange(handler.n_cells, dtype=np.int64), 27)[valid]
    size_of = np.tile(col_size, handler.n_cells)[valid]
    start_of = flat[valid]
    batch_of = _cell_batch_ids(plan, handler.n_cells)[cell_of]

    order = np.argsort(start_of, kind="stable")
    s_sorted = start_of[order]
    head = np.flatnonzero(np.concatenate(([True], s_sorted[1:] != s_sorted[:-1])))
    ent_start = s_sorted[head]
    ent_size = size_of[order][head]
    ent_first = np.minimum.reduceat(batch_of[order], head)
    ent_last = np.maximum.reduceat(batch_of[order], head)

    cmask = np.zeros(n_nodes, dtype=bool)
    if handler.constrained_dofs.size:
        nodes, counts = np.unique(handler.constrained_dofs // comp, return_counts=True)
        if np.any(counts != comp):
            raise ValueError("constraints must cover whole nodes (all components)")
        cmask[nodes] = True
    csum = np.concatenate(([0], np.cumsum(cmask)))
    covered = csum[ent_start + ent_size] - csum[ent_start]
    if np.any((covered > 0) & (covered < ent_size)):
        raise ValueError("partially constrained entity cannot keep contiguous blocks")
    is_con = cmask[ent_start]
    cat = np.where(is_con, 3, np.where(ent_first == ent_last, 0, 1))
    if remote_shared is not None and len(remote_shared):
        rmask = np.zeros(n_nodes, dtype=bool)
        rmask[np.asarray(remote_shared, dtype=np.int64)] = True
        rsum = np.concatenate(([0], np.cumsum(rmask)))
        rcov = rsum[ent_start + ent_size] - rsum[ent_start]
        if np.any((rcov > 0) & (rcov < ent_size)):
            raise ValueError("partially remote-shared entity cannot keep contiguous blocks")
        cat = np.where((rcov > 0) & ~is_con, 2, cat)

    # one composite sort: category, then the category's own three keys
    k1 = np.where(cat == 1, -(ent_first + ent_last), ent_first)
    k2 = np.where(cat == 1, ent_last - ent_first, ent_last)
    seq = np.lexsort((ent_start, k2, k1, cat))
    new_start_sorted = np.cumsum(ent_size[seq]) - ent_size[seq]
    new_start = np.empty_like(ent_start)
    new_start[seq] = new_start_sorted
    if int(ent_size.sum()) != n_nodes:
        raise AssertionError("renumbering did not produce a bijection")

    node_perm = np.empty(n_nodes, dtype=np.int64)
    node_perm[np.repeat(ent_start, ent_size) + _ragged_arange(ent_size)] = \
        np.repeat(new_start, ent_size) + _ragged_arange(ent_size)

    new_blocks = np.full_like(blocks, -1)
    pos = np.searchsorted(ent_start, flat[valid])
    nb_flat = new_blocks.ravel()
    nb_flat[valid] = new_start[pos]
    new_blocks = nb_flat.reshape(blocks.shape)

    perm = (node_perm[:, None] * comp + np.arange(comp)).ravel()
    new_constrained = np.sort(perm[handler.constrained_dofs])
    return DofHandler(handler.n_dofs, comp, p, handler.cells_per_dim, new_blocks,
                      new_constrained, "optimized", perm)


# ---------------------------------------------------------------------------
# range schedule


def compute_range_schedule(handler: DofHandler, plan: BatchPlan) -> RangeSchedule:
    """First/last touching batch of every 64-entry range and per-batch pre/post
    lists; ranges with constrained entries run pre at batch 0 and post at the
    last batch (reference dofs.py:395-423)."""
    n_ranges = -(-handler.n_dofs // RANGE_SIZE)
    nb = plan.n_batches
    first = np.full(n_ranges, nb, dtype=np.int64)
    last = np.full(n_ranges, -1, dtype=np.int64)
    # batches are visited in ascending order, so "first" only needs writes in
    # descending order and "last" in ascending order -- no ufunc.at required
    touched = [np.unique(expand_batch(handler, cells) // RANGE_SIZE) for cells in plan.batches]
    for b in range(nb):
        last[touched[b]] = b
    for b in range(nb - 1, -1, -1):
        first[touched[b]] = b
    hole = first == nb
    first[hole] = 0
    last[hole] = nb - 1
    pre_b, post_b = first.copy(), last.copy()
    if handler.constrained_dofs.size:
        cr = np.unique(handler.constrained_dofs // RANGE_SIZE)
        pre_b[cr] = 0
        post_b[cr] = nb - 1
    pre_sorted = np.argsort(pre_b, kind="stable")
    post_sorted = np.argsort(post_b, kind="stable")
    pre_cut = np.searchsorted(pre_b[pre_sorted], np.arange(nb + 1))
    post_cut = np.searchsorted(post_b[post_sorted], np.arange(nb + 1))
    pre = tuple(pre_sorted[pre_cut[b]:pre_cut[b + 1]] for b in range(nb))
    post = tuple(post_sorted[post_cut[b]:post_cut[b + 1]] for b in range(nb))
    return RangeSchedule(RANGE_SIZE, handler.n_dofs, first, last, pre, post)
