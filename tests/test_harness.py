"""Benchmark harness mirror (reference bench.py): BP table, manufactured right-hand side against
the reference fixture, energy check, RunRecord.  The GPU part solves BP5 / BP3."""
import math

import numpy as np
import pytest

from paper_2205_08909_b200 import harness
from paper_2205_08909_b200.mesh import GeometryVariant


def test_table_and_errors():
    assert set(harness.BENCHMARK_PROBLEMS) == {"BP1", "BP2", "BP3", "BP4", "BP5"}
    bp5 = harness.BENCHMARK_PROBLEMS["BP5"]
    spec = bp5.operator_spec(5)
    assert (spec.n_q_1d, spec.quadrature_kind, spec.equation, spec.components) == (6, "gauss_lobatto", "laplace", 1)
    assert harness.BENCHMARK_PROBLEMS["BP3"].n_quadrature(4) == 6
    with pytest.raises(ValueError):
        harness.assemble_problem("BP9", 2, (2, 2, 2))
    with pytest.raises(NotImplementedError):
        harness.assemble_problem("BP4", 2, (2, 2, 2))
    u = harness.manufactured_solution(np.array([[0.5, 0.5, 0.5], [0.0, 0.3, 0.7]]))
    assert u[0] == pytest.approx(1.0) and abs(u[1]) < 1e-15
    assert harness.manufactured_forcing(np.array([[0.5, 0.5, 0.5]]), "laplace")[0] == pytest.approx(3 * math.pi ** 2)


@pytest.mark.gpu
def test_bp5_energy_and_record():
    """Discrete energy x.b -> 3 pi^2 / 8 (reference tests/test_bench.py:110-121), BP5 on the
    sine-deformed mesh, stored final tensor; and the timing record."""
    from paper_2205_08909_b200.solvers import SolverConfig, solve
    op, b, minv = harness.assemble_problem("BP5", 5, (6, 6, 6))
    res = solve("combined_pcg", op, b, minv=minv, config=SolverConfig(tolerance=1e-10, max_iterations=2000))
    assert res.converged
    assert res.x @ b == pytest.approx(3.0 * math.pi ** 2 / 8.0, rel=1e-3)
    ref = solve("pcg", op, b, minv=minv, config=SolverConfig(tolerance=1e-10, max_iterations=2000))
    assert np.max(np.abs(ref.x - res.x)) < 1e-8
    rec = harness.run_benchmark("BP5", 5, (8, 8, 8), "combined_pcg", iterations=20, repeats=2)
    assert rec.n_dofs == 41 ** 3 and rec.iterations == 20 and rec.throughput > 0
    assert (rec.reads_per_dof, rec.writes_per_dof) == (4.5, 3.5)
    # BP3 (p+2 Gauss points) runs on the affine path
    op3, b3, minv3 = harness.assemble_problem("BP3", 3, (5, 5, 5), geometry=GeometryVariant.AFFINE, deform=0.0)
    r3 = solve("combined_pcg", op3, b3, minv=minv3, config=SolverConfig(tolerance=1e-10, max_iterations=2000))
    assert r3.x @ b3 == pytest.approx(3.0 * math.pi ** 2 / 8.0, rel=1e-3)


def test_manufactured_rhs_matches_reference(golden):
    """build_rhs against the reference's (fixture generated in the authoring container by the
    snippet recorded in oracle/make_golden.py::harness_rhs)."""
    from paper_2205_08909_b200 import dofs, mesh as pm, tensor

    class HostOnly:  # build_rhs needs spec/mesh/handler/quadrature/basis, not the device
        pass

    m = pm.deform_mesh(pm.build_cartesian_mesh((3, 2, 2)), 0.05)
    f = HostOnly()
    f.spec = harness.BENCHMARK_PROBLEMS["BP5"].operator_spec(3)
    f.mesh, f.handler = m, dofs.distribute_dofs(m, 3, 1, True)
    f.quadrature = tensor.gauss_lobatto_quadrature(4)
    f.basis = tensor.lagrange_basis(3, f.quadrature)
    b = harness.build_rhs(f)
    ref = golden["harness"]["bp5_p3_322_rhs"]
    assert np.max(np.abs(b - ref)) / np.max(np.abs(ref)) < 1e-13
