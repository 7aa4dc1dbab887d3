"""Host-side tables of the package against the reference fixtures: integer tables
bit-exact, 1D tables to 1e-15.  CPU only."""
import numpy as np
import pytest

from paper_2205_08909_b200 import dofs, mesh as pmesh, tensor
from _problems import CURVED_CASES, NUMBERING_CASES, host_tables, rel


def test_batch_size_frozen_values(golden):
    # reference tests/test_dofs.py:145-152
    assert [dofs.batch_size(5, 3, 8), dofs.batch_size(5, 1, 8), dofs.batch_size(1, 1, 1),
            dofs.batch_size(3, 1, 8), dofs.batch_size(9, 3, 1)] == [16, 32, 128, 128, 2]
    assert list(golden["numbering"]["batch_sizes"]) == [16, 32, 128, 128, 2]


@pytest.mark.parametrize("cells,p", NUMBERING_CASES)
def test_numbering_bit_exact(golden, cells, p):
    g = golden["numbering"]
    tag = "x".join(map(str, cells)) + f"_p{p}"
    m = pmesh.build_cartesian_mesh(cells)
    h = dofs.distribute_dofs(m, p, 1, constrain_boundary=True)
    assert h.n_dofs == np.prod([c * p + 1 for c in cells])
    assert h.cell_index_blocks.dtype == np.int32
    assert np.array_equal(h.cell_index_blocks, g[f"{tag}_blocks"])
    assert np.array_equal(h.constrained_dofs, g[f"{tag}_constrained"])
    for trav in ("morton", "lexicographic"):
        plan = dofs.make_batches(m, int(g[f"{tag}_{trav}_bsize"][0]), trav)
        assert np.array_equal(np.concatenate(plan.batches), g[f"{tag}_{trav}_order"])
        r = dofs.renumber_optimized(h, plan)
        assert np.array_equal(r.cell_index_blocks, g[f"{tag}_{trav}_rblocks"])
        assert np.array_equal(r.permutation, g[f"{tag}_{trav}_perm"])
        assert np.array_equal(r.constrained_dofs, g[f"{tag}_{trav}_rconstrained"])
        s = dofs.compute_range_schedule(r, plan)
        assert np.array_equal(s.first_touch_batch, g[f"{tag}_{trav}_first"])
        assert np.array_equal(s.last_touch_batch, g[f"{tag}_{trav}_last"])
        # permutation is a bijection, constrained DoFs form the tail (tests/test_dofs.py:205-221)
        assert np.array_equal(np.sort(r.permutation), np.arange(h.n_dofs))
        k = len(r.constrained_dofs)
        assert np.array_equal(r.constrained_dofs, np.arange(h.n_dofs - k, h.n_dofs))
        with pytest.raises(ValueError):
            dofs.renumber_optimized(r, plan)


def test_morton_small_cases():
    # reference tests/test_dofs.py:178-198
    m = pmesh.build_cartesian_mesh((2, 2, 2))
    assert list(dofs.make_batches(m, 8, "morton").batches[0]) == [0, 1, 2, 3, 4, 5, 6, 7]
    m = pmesh.build_cartesian_mesh((3, 4, 2))
    order = np.concatenate(dofs.make_batches(m, 5, "morton").batches)
    assert sorted(order) == list(range(24)) and list(order[:4]) == [0, 1, 3, 4]


def test_shared_face_hand_case():
    # reference tests/test_dofs.py:240-260: two p=1 cells, one per batch: shared face -> {8..11}
    m = pmesh.build_cartesian_mesh((2, 1, 1))
    h = dofs.distribute_dofs(m, 1)
    r = dofs.renumber_optimized(h, dofs.make_batches(m, 1))
    shared = np.intersect1d(dofs.expand_cell_indices(r, 0), dofs.expand_cell_indices(r, 1))
    assert list(shared) == [8, 9, 10, 11]


def test_errors_like_reference():
    m = pmesh.build_cartesian_mesh((2, 2, 2))
    with pytest.raises(ValueError):
        dofs.distribute_dofs(m, 0)
    with pytest.raises(ValueError):
        dofs.distribute_dofs(m, 2, components=2)
    with pytest.raises(ValueError):
        dofs.make_batches(m, 0)
    with pytest.raises(ValueError):
        dofs.make_batches(m, 2, "hilbert")
    with pytest.raises(IndexError):
        dofs.expand_cell_indices(dofs.distribute_dofs(m, 2), 8)
    with pytest.raises(ValueError):
        pmesh.build_cartesian_mesh((0, 1, 1))
    with pytest.raises(ValueError):
        pmesh.deform_mesh(pmesh.build_cartesian_mesh((1, 1, 1)), 0.9)
    with pytest.raises(ValueError):
        pmesh.precompute_geometry(pmesh.deform_mesh(m, 0.05), pmesh.GeometryVariant.AFFINE,
                                  tensor.gauss_quadrature(3))


def test_1d_tables(golden):
    g = golden["tables"]
    for n in range(1, 11):
        q = tensor.gauss_quadrature(n)
        assert np.allclose(q.points, g[f"gauss_x_{n}"], rtol=0, atol=1e-15)
        assert np.allclose(q.weights, g[f"gauss_w_{n}"], rtol=0, atol=1e-15)
        if n >= 2:
            q = tensor.gauss_lobatto_quadrature(n)
            assert np.allclose(q.points, g[f"gl_x_{n}"], rtol=0, atol=1e-15)
            assert np.allclose(q.weights, g[f"gl_w_{n}"], rtol=0, atol=1e-15)
    for p in range(1, 9):
        for nq in (p + 1, p + 2):
            b = tensor.lagrange_basis(p, tensor.gauss_quadrature(nq))
            assert np.allclose(b.shape_values, g[f"S_{p}_{nq}"], rtol=0, atol=2e-15)
            assert rel(b.shape_gradients, g[f"D_{p}_{nq}"]) < 5e-15
            # partition of unity / derivative sums to zero (tests/test_tensor.py:169-174)
            assert np.allclose(b.shape_values.sum(1), 1.0, atol=1e-14)
            assert np.allclose(b.shape_gradients.sum(1), 0.0, atol=1e-12)
            assert np.allclose(b.collocation_gradient @ b.shape_values, b.shape_gradients, atol=1e-12)


def test_quadrature_exactness():
    # reference tests/test_tensor.py:126-145
    for n in range(1, 13):
        q = tensor.gauss_quadrature(n)
        for d in range(2 * n):
            assert q.weights @ q.points ** d == pytest.approx(1.0 / (d + 1), abs=1e-13)
        if n >= 2:
            q = tensor.gauss_lobatto_quadrature(n)
            for d in range(2 * n - 2):
                assert q.weights @ q.points ** d == pytest.approx(1.0 / (d + 1), abs=1e-13)


@pytest.mark.parametrize("ci", range(len(CURVED_CASES)))
def test_host_geometry_matches_reference(golden, ci):
    cells, p, nq, amp = CURVED_CASES[ci]
    g = golden["curved"]
    m, h, plan = host_tables(cells, p, deform=amp)
    quad = tensor.gauss_quadrature(nq)
    ft = pmesh.precompute_geometry(m, pmesh.GeometryVariant.FINAL_TENSOR_LOAD, quad)
    assert ft.doubles_per_cell == 7 * nq ** 3
    assert rel(ft.payload["final_tensor"], g[f"k{ci}_final_tensor"]) < 1e-12
    ij = pmesh.precompute_geometry(m, pmesh.GeometryVariant.INVERSE_JACOBIAN_LOAD, quad)
    assert ij.doubles_per_cell == 10 * nq ** 3
    assert rel(ij.payload["inverse_jacobian"], g[f"k{ci}_inverse_jacobian"]) < 1e-12
    assert rel(ij.payload["jxw"], g[f"k{ci}_jxw"]) < 1e-12
    qc = pmesh.precompute_geometry(m, pmesh.GeometryVariant.QUADRATIC_COMPUTE, quad)
    assert qc.doubles_per_cell == 81 and qc.payload["nodes"].shape == (m.n_cells, 27, 3)


def test_mesh_layout_and_text_roundtrip():
    # reference tests/test_mesh.py:86-145, 329-343
    m = pmesh.build_cartesian_mesh((2, 3, 4), (1.0, 2.0, 3.0))
    assert m.vertex_coordinates.shape == (3 * 4 * 5, 3) and m.cell_vertex_indices.shape == (24, 8)
    assert list(m.cell_vertex_indices[0]) == [0, 1, 3, 4, 12, 13, 15, 16]
    d = pmesh.deform_mesh(m, 0.1)
    centre = np.array([[0.5, 1.0, 1.5]])
    assert np.allclose(d.map_points(centre) - centre, 0.1)
    face = np.array([[0.0, 0.7, 1.1]])
    assert np.allclose(d.map_points(face), face)
    back = pmesh.mesh_from_text(pmesh.mesh_to_text(d))
    assert back.cells_per_dim == d.cells_per_dim and back.deformation == d.deformation


def test_three_component_numbering_matches_reference(golden):
    """distribute_dofs / renumber_optimized with components = 3 (reference dofs.py:138-179, 304-388)."""
    from _problems import VECTOR_CASES
    g = golden["vector3"]
    for ci, (cells, p, nq, numbering, amp, variant) in enumerate(VECTOR_CASES):
        m, h, plan = host_tables(cells, p, numbering=numbering, deform=amp, components=3)
        assert h.components == 3 and h.n_dofs == 3 * int(np.prod([c * p + 1 for c in cells]))
        assert np.array_equal(h.cell_index_blocks, g[f"v{ci}_blocks"])
        assert np.array_equal(h.constrained_dofs, g[f"v{ci}_constrained"])
        if numbering == "optimized":
            assert np.array_equal(h.permutation, g[f"v{ci}_permutation"])


@pytest.mark.parametrize("n", [32, 48])
def test_large_integer_tables_sha256(n):
    """The vectorised numbering / renumbering / schedule at 32^3 and 48^3 cells Q5 (4.2e6 / 1.4e7 DoFs) against
    SHA-256 digests of the reference's tables (tests/golden/big_tables.json, oracle/make_golden.py::
    big_table_digests): bit-exact far beyond the 8^3 meshes whose arrays are committed."""
    import hashlib
    import json
    from pathlib import Path
    ref = json.loads((Path(__file__).parent / "golden" / "big_tables.json").read_text())[str(n)]

    def dg(a):
        a = np.ascontiguousarray(a)
        return hashlib.sha256(a.tobytes()).hexdigest() + f":{a.dtype}:{a.shape}"

    mesh = pmesh.build_cartesian_mesh((n, n, n))
    h = dofs.distribute_dofs(mesh, 5, 1, constrain_boundary=True)
    plan = dofs.make_batches(mesh, dofs.batch_size(5, 1, 8), "morton")
    assert h.n_dofs == ref["n_dofs"]
    assert dg(h.cell_index_blocks) == ref["blocks"]
    assert dg(h.constrained_dofs) == ref["constrained"]
    assert dg(np.concatenate([np.asarray(b) for b in plan.batches])) == ref["batches"]
    hr = dofs.renumber_optimized(h, plan)
    assert dg(hr.cell_index_blocks) == ref["ren_blocks"]
    assert dg(hr.permutation) == ref["ren_permutation"]
    assert dg(hr.constrained_dofs) == ref["ren_constrained"]
    sch = dofs.compute_range_schedule(hr, plan)
    assert dg(sch.first_touch_batch) == ref["schedule_first"]
    assert dg(sch.last_touch_batch) == ref["schedule_last"]
