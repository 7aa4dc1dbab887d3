"""Liveliness reporting: the reference's report on the reference's
schedule, and the same report on the brick schedule the library really uses."""
import numpy as np
import pytest

from paper_2205_08909_b200 import dofs, locality
from _problems import gpu_operator, host_tables


@pytest.mark.parametrize("ci,cells,p", [(0, (8, 8, 8), 4), (1, (6, 5, 4), 5)])
def test_liveliness_matches_reference(golden, ci, cells, p):
    g = golden["locality"]
    for numbering in ("default", "optimized"):
        m, h, plan = host_tables(cells, p, numbering=numbering)
        rep = locality.liveliness(dofs.compute_range_schedule(h, plan))
        key = f"l{ci}_{numbering}"
        assert np.array_equal(rep.distances, g[key + "_distances"])
        assert np.array_equal(rep.cdf_distances, g[key + "_cdf_distances"])
        assert np.array_equal(rep.cdf_fractions, g[key + "_cdf_fractions"])
        nb, same, nr = g[key + "_scalars"]
        assert (rep.n_batches, rep.n_ranges) == (int(nb), int(nr)) and rep.same_batch_fraction == same
        # step-function CDF (reference locality.py:207-213)
        assert rep.fraction_within(-1) == 0.0 and rep.fraction_within(rep.cdf_distances[-1]) == 1.0


def test_measured_transfer_reads_profile():
    t = locality.measured_transfer()
    assert t["bytes_per_dof_model"] == 64.0
    assert 30.0 < t["bytes_per_dof_measured"] < 80.0 and len(t["bytes_per_dof_by_launch"]) == 2


@pytest.mark.gpu
def test_brick_schedule_properties():
    p = 5
    m, h, plan = host_tables((9, 8, 20), p)
    op = gpu_operator(m, h, plan, p, p + 1)
    info = op.info()
    sch = locality.brick_schedule(op)
    rep = locality.liveliness(sch)
    assert rep.n_batches == info["n_bricks"] and sch.n_dofs == h.n_dofs
    assert np.all(sch.first_touch_batch <= sch.last_touch_batch) and sch.first_touch_batch.min() == 0
    # ranges made only of brick-interior DoFs live inside one brick
    n_int_ranges = info["n_interior"] // dofs.RANGE_SIZE
    assert np.all(rep.distances[:n_int_ranges - info["n_bricks"]] <= 1)
    assert rep.same_batch_fraction > 0.8 * info["n_interior"] / h.n_dofs
    assert sum(len(a) for a in sch.pre_schedule) == sch.n_ranges == sum(len(a) for a in sch.post_schedule)
    # one brick: everything is produced and finished in it
    m1, h1, plan1 = host_tables((2, 2, 2), 3)
    rep1 = locality.liveliness(locality.brick_schedule(gpu_operator(m1, h1, plan1, 3, 4, brick=(2, 2, 2))))
    assert rep1.n_batches == 1 and rep1.same_batch_fraction == 1.0
