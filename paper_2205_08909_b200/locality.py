"""Liveliness reporting for the brick schedule.

The reference reports, per 64-entry vector range, how many cell batches lie
between its first and last touch during one operator application
(``locality.py:195-227``, CLI ``liveliness``, ``cli.py:209-228``), and replays a
recorded access trace through an LRU model to predict memory transfer
(``cachesweep``).  On the GPU the batches are bricks and the vector is stored in
the library's brick numbering, so

* :func:`liveliness` is the reference's function on a ``RangeSchedule``;
* :func:`brick_schedule` builds that schedule for the numbering and launch order
  the library really uses (from the device permutation, not from a model);
* :func:`measured_transfer` stands in for the cache replay: it reads the DRAM
  bytes per DoF and iteration that ncu measured for the fused kernel
  (``profiles/traffic.json``) and sets them beside the model figure.

Host-side reporting only; nothing here is on the hot path.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .dofs import RANGE_SIZE, RangeSchedule, _expand_scalar

__all__ = ["LivelinessReport", "liveliness", "brick_schedule", "measured_transfer"]


@dataclass(frozen=True)
class LivelinessReport:
    """Field for field the reference's report (locality.py:195-213)."""

    distances: np.ndarray
    n_batches: int
    same_batch_fraction: float
    cdf_distances: np.ndarray
    cdf_fractions: np.ndarray

    @property
    def n_ranges(self) -> int:
        return len(self.distances)

    def fraction_within(self, distance) -> np.ndarray:
        idx = np.searchsorted(self.cdf_distances, np.asarray(distance), side="right")
        return np.concatenate([[0.0], self.cdf_fractions])[idx]


def liveliness(schedule: RangeSchedule) -> LivelinessReport:
    """Batches between first and last touch of every range (locality.py:216-227)."""
    first = np.asarray(schedule.first_touch_batch)
    last = np.asarray(schedule.last_touch_batch)
    distances = last - first
    n_batches = int(last.max()) + 1 if len(last) else 1
    uniq, counts = np.unique(distances, return_counts=True)
    return LivelinessReport(distances, n_batches, float(np.mean(distances == 0)), uniq,
                            np.cumsum(counts) / len(distances))


def brick_schedule(op, chunk: int = 1 << 15) -> RangeSchedule:
    """First / last touching brick of every 64-entry range of one component
    field in the library's brick numbering; bricks count in launch order (x
    fastest).  Same container as ``compute_range_schedule`` (dofs.py:395-423):
    the pre list of a brick holds the ranges it is the first to touch."""
    info = op.info()
    bx, by, bz = info["brick"]
    nx, ny, nz = op.mesh.cells_per_dim
    mbx, mby = -(-nx // bx), -(-ny // by)
    n_bricks = int(info["n_bricks"])
    perm = op.device_permutation().astype(np.int64)
    n_nodes = len(perm)
    n_ranges = -(-n_nodes // RANGE_SIZE)
    first = np.full(n_ranges, n_bricks, dtype=np.int64)
    last = np.full(n_ranges, -1, dtype=np.int64)
    for lo in range(0, op.mesh.n_cells, chunk):
        cells = np.arange(lo, min(lo + chunk, op.mesh.n_cells))
        cx, cy, cz = cells % nx, (cells // nx) % ny, cells // (nx * ny)
        brick = (cx // bx) + mbx * ((cy // by) + mby * (cz // bz))
        ranges = perm[_expand_scalar(op.handler, cells)] // RANGE_SIZE
        b = np.broadcast_to(brick[:, None], ranges.shape)
        np.minimum.at(first, ranges.ravel(), b.ravel())
        np.maximum.at(last, ranges.ravel(), b.ravel())
    order_f = np.argsort(first, kind="stable")
    order_l = np.argsort(last, kind="stable")
    cut_f = np.searchsorted(first[order_f], np.arange(n_bricks + 1))
    cut_l = np.searchsorted(last[order_l], np.arange(n_bricks + 1))
    pre = tuple(order_f[cut_f[b]:cut_f[b + 1]] for b in range(n_bricks))
    post = tuple(order_l[cut_l[b]:cut_l[b + 1]] for b in range(n_bricks))
    return RangeSchedule(RANGE_SIZE, n_nodes, first, last, pre, post)


def measured_transfer(profile: str | Path = None) -> dict:
    """Measured DRAM bytes per DoF and merged iteration of the fused kernel next
    to the model (the GPU stand-in for the reference's ``cachesweep`` table)."""
    path = Path(profile) if profile else Path(__file__).resolve().parent.parent / "profiles" / "traffic.json"
    t = json.loads(path.read_text())
    n = float(t["k_brick_merged_bytes_per_launch"]) / float(t["bytes_per_dof"])
    per_launch = [b / n for b in t["launches"]]
    return {"workload": t["workload"], "bytes_per_dof_measured": float(t["bytes_per_dof"]),
            "bytes_per_dof_by_launch": per_launch, "bytes_per_dof_model": 64.0,
            "source": t["source"]}
