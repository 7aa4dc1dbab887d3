"""Generate tests/golden/*.npz by running the UNMODIFIED reference.

Run in the authoring container only (needs /root/reference):
    python oracle/make_golden.py
The fixtures are committed; nothing at test time on the GPU box reads
/root/reference.  Inputs are seeded (numpy default_rng), so the script is
reproducible.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from mfcg.dofs import (batch_size, compute_range_schedule, distribute_dofs,  # noqa: E402
                       make_batches, renumber_optimized)
from mfcg.mesh import GeometryVariant, build_cartesian_mesh, deform_mesh, precompute_geometry  # noqa: E402
from mfcg.operator import MatrixFreeOperator, OperatorSpec  # noqa: E402
from mfcg.solvers import SolverConfig, solve  # noqa: E402
from mfcg.tensor import gauss_lobatto_quadrature, gauss_quadrature, lagrange_basis  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
OUT.mkdir(parents=True, exist_ok=True)


def build(cells, p, nq, *, constrain=True, numbering="default", traversal="morton", batch=None,
          deform=0.0, variant=GeometryVariant.AFFINE, quadrature="gauss", components=1):
    mesh = build_cartesian_mesh(cells)
    if deform:
        mesh = deform_mesh(mesh, deform)
    h = distribute_dofs(mesh, p, components, constrain_boundary=constrain)
    plan = make_batches(mesh, batch or batch_size(p, components, 8), traversal)
    if numbering == "optimized":
        h = renumber_optimized(h, plan)
    spec = OperatorSpec("laplace", components, p, nq, variant, quadrature)
    return MatrixFreeOperator(spec, mesh, h, plan), h, plan, mesh


def hist_array(res):
    return np.array([[e["alpha"], e["beta"], e["gamma"], e["residual"]] for e in res.history])


def tables():
    out = {}
    for n in range(1, 11):
        q = gauss_quadrature(n)
        out[f"gauss_x_{n}"], out[f"gauss_w_{n}"] = q.points, q.weights
        if n >= 2:
            q = gauss_lobatto_quadrature(n)
            out[f"gl_x_{n}"], out[f"gl_w_{n}"] = q.points, q.weights
    for p in range(1, 9):
        for nq in (p + 1, p + 2):
            b = lagrange_basis(p, gauss_quadrature(nq))
            out[f"S_{p}_{nq}"], out[f"D_{p}_{nq}"] = b.shape_values, b.shape_gradients
        b = lagrange_basis(p, gauss_lobatto_quadrature(p + 1))
        out[f"Dgl_{p}"] = b.shape_gradients
    np.savez_compressed(OUT / "tables.npz", **out)


NUMBERING_CASES = [
    ((2, 2, 2), 1), ((2, 1, 1), 1), ((3, 4, 2), 2), ((2, 2, 2), 3), ((5, 3, 6), 5),
    ((8, 8, 8), 4), ((4, 4, 4), 5), ((6, 6, 6), 1), ((7, 6, 5), 4),
]


def numbering():
    out = {}
    for cells, p in NUMBERING_CASES:
        tag = "x".join(map(str, cells)) + f"_p{p}"
        mesh = build_cartesian_mesh(cells)
        h = distribute_dofs(mesh, p, 1, constrain_boundary=True)
        out[f"{tag}_blocks"] = h.cell_index_blocks
        out[f"{tag}_constrained"] = h.constrained_dofs
        for trav in ("morton", "lexicographic"):
            plan = make_batches(mesh, batch_size(p, 1, 8) if trav == "morton" else 3, trav)
            out[f"{tag}_{trav}_order"] = np.concatenate(plan.batches)
            out[f"{tag}_{trav}_bsize"] = np.array([plan.batch_size])
            r = renumber_optimized(h, plan)
            out[f"{tag}_{trav}_rblocks"] = r.cell_index_blocks
            out[f"{tag}_{trav}_perm"] = r.permutation
            out[f"{tag}_{trav}_rconstrained"] = r.constrained_dofs
            s = compute_range_schedule(r, plan)
            out[f"{tag}_{trav}_first"] = s.first_touch_batch
            out[f"{tag}_{trav}_last"] = s.last_touch_batch
    out["batch_sizes"] = np.array([batch_size(5, 3, 8), batch_size(5, 1, 8), batch_size(1, 1, 1),
                                   batch_size(3, 1, 8), batch_size(9, 3, 1)])
    np.savez_compressed(OUT / "numbering.npz", **out)


# (cells, p, nq, numbering, constrain)
APPLY_CASES = [
    ((2, 2, 2), 3, 4, "default", True),
    ((3, 4, 2), 2, 3, "default", True),
    ((2, 3, 2), 1, 2, "default", True),
    ((4, 4, 4), 5, 6, "optimized", True),
    ((5, 4, 9), 5, 6, "default", True),
    ((9, 5, 3), 5, 7, "optimized", True),
    ((3, 3, 3), 7, 8, "default", True),
    ((2, 3, 2), 8, 9, "default", True),
    ((7, 6, 5), 4, 5, "optimized", True),
    ((11, 7, 3), 3, 4, "default", True),
    ((4, 3, 5), 6, 7, "default", True),
    ((3, 3, 2), 4, 5, "default", False),
    ((21, 12, 2), 2, 3, "default", True),
    ((18, 17, 3), 1, 2, "optimized", True),
]


def apply_cases():
    out = {}
    for ci, (cells, p, nq, numb, con) in enumerate(APPLY_CASES):
        op, h, plan, mesh = build(cells, p, nq, constrain=con, numbering=numb)
        rng = np.random.default_rng(100 + ci)
        u = rng.standard_normal(h.n_dofs)
        out[f"c{ci}_u"] = u
        out[f"c{ci}_Au"] = op.apply(u)
        out[f"c{ci}_invdiag"] = op.compute_diagonal().inverse_diagonal
        out[f"c{ci}_blocks"] = h.cell_index_blocks
        out[f"c{ci}_constrained"] = h.constrained_dofs
    np.savez_compressed(OUT / "apply.npz", **out)


def config1():
    """BASELINE.json configs[0]: 8^3 cells, Q4, 5-point Gauss, 100 fixed iterations."""
    op, h, plan, mesh = build((8, 8, 8), 4, 5)
    minv = op.compute_diagonal()
    b = np.random.default_rng(0).uniform(-1.0, 1.0, h.n_dofs)
    b[h.constrained_dofs] = 0.0
    out = {"b": b, "invdiag": minv.inverse_diagonal, "Ab": op.apply(b)}
    cfg = SolverConfig(fixed_iterations=100)
    for variant in ("pcg", "combined_pcg", "cg", "combined_cg"):
        res = solve(variant, op, b, minv=minv, config=cfg)
        out[f"{variant}_hist"] = hist_array(res)
        out[f"{variant}_x"] = res.x
    # the reference's own re-ordering envelope: same maths, lexicographic batches
    op2, h2, _, _ = build((8, 8, 8), 4, 5, traversal="lexicographic", batch=7)
    for variant in ("pcg", "combined_pcg"):
        res = solve(variant, op2, b, minv=op2.compute_diagonal(), config=cfg)
        out[f"{variant}_hist_reordered"] = hist_array(res)
        out[f"{variant}_x_reordered"] = res.x
    # tolerance-terminated run (early exit semantics)
    for variant in ("pcg", "combined_pcg"):
        res = solve(variant, op, b, minv=minv, config=SolverConfig(tolerance=1e-6, max_iterations=500))
        out[f"{variant}_tol_hist"] = hist_array(res)
        out[f"{variant}_tol_iters"] = np.array([res.iterations, int(res.converged)])
    np.savez_compressed(OUT / "config1.npz", **out)


def q5_small():
    """BASELINE.json configs[1], smallest rungs (4^3 and 6^3 cells, Q5), 200 iterations, plus
    optimized numbering for 4^3."""
    out = {}
    for n, numb in ((4, "default"), (6, "default"), (4, "optimized")):
        op, h, plan, mesh = build((n, n, n), 5, 6, numbering=numb)
        minv = op.compute_diagonal()
        b = np.random.default_rng(0).uniform(-1.0, 1.0, h.n_dofs)
        if numb == "optimized":
            bo = np.empty_like(b)
            bo[h.permutation] = b
            b = bo
        b[h.constrained_dofs] = 0.0
        tag = f"n{n}_{numb}"
        out[f"{tag}_b"] = b
        for variant in ("pcg", "combined_pcg"):
            res = solve(variant, op, b, minv=minv, config=SolverConfig(fixed_iterations=200))
            out[f"{tag}_{variant}_hist"] = hist_array(res)
            out[f"{tag}_{variant}_x"] = res.x
    np.savez_compressed(OUT / "q5_small.npz", **out)


CURVED_CASES = [((3, 3, 3), 3, 4, 0.1), ((4, 3, 5), 5, 6, 0.1), ((2, 2, 2), 2, 4, 0.05)]


def curved():
    out = {}
    for ci, (cells, p, nq, amp) in enumerate(CURVED_CASES):
        op, h, plan, mesh = build(cells, p, nq, deform=amp, variant=GeometryVariant.FINAL_TENSOR_LOAD)
        rng = np.random.default_rng(200 + ci)
        u = rng.standard_normal(h.n_dofs)
        out[f"k{ci}_u"] = u
        out[f"k{ci}_Au"] = op.apply(u)
        out[f"k{ci}_invdiag"] = op.compute_diagonal().inverse_diagonal
        out[f"k{ci}_final_tensor"] = op.geometry.payload["final_tensor"]
        g2 = precompute_geometry(mesh, GeometryVariant.INVERSE_JACOBIAN_LOAD, op.quadrature)
        out[f"k{ci}_inverse_jacobian"] = g2.payload["inverse_jacobian"]
        out[f"k{ci}_jxw"] = g2.payload["jxw"]
        b = np.random.default_rng(0).uniform(-1.0, 1.0, h.n_dofs)
        b[h.constrained_dofs] = 0.0
        res = solve("combined_pcg", op, b, minv=op.compute_diagonal(), config=SolverConfig(fixed_iterations=40))
        out[f"k{ci}_b"] = b
        out[f"k{ci}_combined_pcg_hist"] = hist_array(res)
        out[f"k{ci}_combined_pcg_x"] = res.x
    np.savez_compressed(OUT / "curved.npz", **out)


def harness_rhs():
    """Manufactured right-hand sides: BP5 and BP4 (3 components), p = 3, (3,2,2) cells,
    deformation 0.05."""
    from mfcg.bench import assemble_problem
    _, b, _ = assemble_problem("BP5", 3, (3, 2, 2))
    _, b4, _ = assemble_problem("BP4", 3, (3, 2, 2))
    np.savez_compressed(OUT / "harness.npz", bp5_p3_322_rhs=b, bp4_p3_322_rhs=b4)


# (cells, p, nq, numbering, deformation, geometry variant): 3-component Laplace (BP4-type)
VECTOR_CASES = [((3, 2, 2), 2, 3, "default", 0.0, "affine"),
                ((4, 4, 4), 5, 6, "optimized", 0.0, "affine"),
                ((3, 3, 3), 3, 4, "default", 0.1, "final_tensor_load"),
                ((5, 4, 3), 4, 5, "default", 0.0, "affine")]


def vector3():
    out = {}
    for ci, (cells, p, nq, numbering, amp, variant) in enumerate(VECTOR_CASES):
        op, h, plan, mesh = build(cells, p, nq, numbering=numbering, deform=amp,
                                  variant=GeometryVariant(variant), components=3)
        rng = np.random.default_rng(300 + ci)
        u = rng.standard_normal(h.n_dofs)
        out[f"v{ci}_blocks"] = h.cell_index_blocks
        out[f"v{ci}_constrained"] = h.constrained_dofs
        if h.permutation is not None:
            out[f"v{ci}_permutation"] = h.permutation
        out[f"v{ci}_u"] = u
        out[f"v{ci}_Au"] = op.apply(u)
        minv = op.compute_diagonal()
        out[f"v{ci}_invdiag"] = minv.inverse_diagonal
        b = np.random.default_rng(0).uniform(-1.0, 1.0, h.n_dofs)
        if h.permutation is not None:
            bo = np.empty_like(b)
            bo[h.permutation] = b
            b = bo
        b[h.constrained_dofs] = 0.0
        out[f"v{ci}_b"] = b
        for variant_name in ("pcg", "combined_pcg", "combined_cg"):
            res = solve(variant_name, op, b, minv=None if variant_name == "combined_cg" else minv,
                        config=SolverConfig(fixed_iterations=30))
            out[f"v{ci}_{variant_name}_hist"] = hist_array(res)
            out[f"v{ci}_{variant_name}_x"] = res.x
    np.savez_compressed(OUT / "vector3.npz", **out)


def locality():
    """Liveliness reports of the reference (locality.py:216-227) for config 1 and a Q5 mesh."""
    from mfcg.locality import liveliness
    out = {}
    for ci, (cells, p) in enumerate([((8, 8, 8), 4), ((6, 5, 4), 5)]):
        for numbering in ("default", "optimized"):
            op, h, plan, mesh = build(cells, p, p + 1, numbering=numbering)
            rep = liveliness(compute_range_schedule(h, plan))
            key = f"l{ci}_{numbering}"
            out[key + "_distances"] = rep.distances
            out[key + "_cdf_distances"] = rep.cdf_distances
            out[key + "_cdf_fractions"] = rep.cdf_fractions
            out[key + "_scalars"] = np.array([rep.n_batches, rep.same_batch_fraction, rep.n_ranges])
    np.savez_compressed(OUT / "locality.npz", **out)


def bp_canonical():
    """BP3 / BP4 exactly as the reference's harness builds them (bench.py:153-187 defaults: sine-deformed mesh
    0.05, final_tensor_load, n_q = p + 2): manufactured RHS, one apply, the Jacobi diagonal, 25 iterations of
    pcg and combined_pcg."""
    from mfcg.bench import assemble_problem
    out = {}
    for key, (bp, p, cells) in {"bp3": ("BP3", 5, (3, 3, 3)), "bp4": ("BP4", 5, (2, 2, 3)),
                                "bp3_p2": ("BP3", 2, (4, 3, 5))}.items():
        op, b, minv = assemble_problem(bp, p, cells)
        assert op.spec.n_q_1d == p + 2 and op.mesh.deformation == 0.05
        u = np.random.default_rng(17).standard_normal(op.n_dofs)
        out[f"{key}_b"] = b
        out[f"{key}_u"] = u
        out[f"{key}_Au"] = op.apply(u)
        out[f"{key}_invdiag"] = minv.inverse_diagonal
        for variant_name in ("pcg", "combined_pcg"):
            res = solve(variant_name, op, b, minv=minv, config=SolverConfig(fixed_iterations=25))
            out[f"{key}_{variant_name}_hist"] = hist_array(res)
            out[f"{key}_{variant_name}_x"] = res.x
    np.savez_compressed(OUT / "bp_canonical.npz", **out)


def big_table_digests():
    """SHA-256 of the reference's integer tables on meshes too large to commit as arrays (32^3 and 48^3 cells,
    Q5): block table, renumbering (blocks, permutation, constrained tail), Dirichlet set, range schedule
    first/last, Morton batches.  The package's vectorised tables must reproduce the digests bit for bit."""
    import hashlib
    import json

    def dg(a):
        a = np.ascontiguousarray(a)
        return hashlib.sha256(a.tobytes()).hexdigest() + f":{a.dtype}:{a.shape}"

    out = {}
    for n in (32, 48):
        mesh = build_cartesian_mesh((n, n, n))
        h = distribute_dofs(mesh, 5, 1, constrain_boundary=True)
        plan = make_batches(mesh, batch_size(5, 1, 8), "morton")
        hr = renumber_optimized(h, plan)
        sch = compute_range_schedule(hr, plan)
        out[str(n)] = {
            "n_dofs": int(h.n_dofs),
            "blocks": dg(h.cell_index_blocks), "constrained": dg(h.constrained_dofs),
            "batches": dg(np.concatenate([np.asarray(b) for b in plan.batches])),
            "ren_blocks": dg(hr.cell_index_blocks), "ren_permutation": dg(hr.permutation),
            "ren_constrained": dg(hr.constrained_dofs),
            "schedule_first": dg(sch.first_touch_batch), "schedule_last": dg(sch.last_touch_batch),
        }
        print("digests", n, out[str(n)]["n_dofs"], flush=True)
    (OUT / "big_tables.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    import sys as _sys
    if len(_sys.argv) > 1:  # regenerate selected fixtures only: python oracle/make_golden.py bp_canonical ...
        for name in _sys.argv[1:]:
            globals()[name]()
        raise SystemExit(0)
    tables()
    harness_rhs()
    numbering()
    apply_cases()
    config1()
    q5_small()
    curved()
    vector3()
    locality()
    bp_canonical()
    big_table_digests()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
