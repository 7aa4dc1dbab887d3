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
        harness.assemble_problem("BP2", 2, (2, 2, 2))      # mass operators are out of scope
    assert harness.BENCHMARK_PROBLEMS["BP4"].operator_spec(3).components == 3
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
    # BP4: three components, each carrying the same manufactured problem -> three times the energy
    op4, b4, minv4 = harness.assemble_problem("BP4", 3, (5, 5, 5), geometry=GeometryVariant.AFFINE, deform=0.0)
    assert op4.n_dofs == 3 * 16 ** 3 and np.array_equal(b4[0::3], b3) and np.array_equal(b4[2::3], b3)
    r4 = solve("combined_pcg", op4, b4, minv=minv4, config=SolverConfig(tolerance=1e-10, max_iterations=2000))
    assert r4.converged and r4.x @ b4 == pytest.approx(9.0 * math.pi ** 2 / 8.0, rel=1e-3)
    assert np.max(np.abs(r4.x[1::3] - r3.x)) < 1e-8
    rec4 = harness.run_benchmark("BP4", 3, (5, 5, 5), "combined_pcg", iterations=10, repeats=1,
                                 geometry=GeometryVariant.AFFINE, deform=0.0)
    assert rec4.n_dofs == 3 * 16 ** 3 and rec4.iterations == 10


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
    # BP4: p + 2 Gauss points, three interleaved components (reference bench.py:113-116)
    f.spec = harness.BENCHMARK_PROBLEMS["BP4"].operator_spec(3)
    f.handler = dofs.distribute_dofs(m, 3, 3, True)
    f.quadrature = tensor.gauss_quadrature(5)
    f.basis = tensor.lagrange_basis(3, f.quadrature)
    b4 = harness.build_rhs(f)
    ref4 = golden["harness"]["bp4_p3_322_rhs"]
    assert b4.shape == ref4.shape and np.max(np.abs(b4 - ref4)) / np.max(np.abs(ref4)) < 1e-13


def test_bench_csv_schema_matches_reference():
    """Header and field formatting of the reference's `mfcg bench` CSV (cli.py:155-186): `repr` wall time,
    %.6g floats, cells joined with x."""
    from paper_2205_08909_b200 import harness as H
    rec = H.RunRecord.from_run("BP5", 5, (4, 4, 4), 9261, "combined_pcg", 100, 0.0123456789, 1.5e-7)
    text = H.write_bench_csv([rec])
    head, row = text.strip().split("\n")
    assert head == ("bp,degree,cells,n_dofs,variant,iterations,wall_time_s,throughput_dofs_per_s,final_residual,"
                    "model_reads_per_dof,model_writes_per_dof")
    f = row.split(",")
    assert f[:6] == ["BP5", "5", "4x4x4", "9261", "combined_pcg", "100"]
    assert f[6] == repr(0.0123456789) and f[7] == f"{9261 * 100 / 0.0123456789:.6g}" and f[8] == "1.5e-07"
    assert [float(f[9]), float(f[10])] == [rec.reads_per_dof, rec.writes_per_dof]
