"""Shared builders: the same seeded problem as (a) host tables from the package,
(b) an oracle `Problem`, (c) a GPU operator.  The case lists mirror
oracle/make_golden.py."""
import numpy as np

from paper_2205_08909_b200 import dofs, mesh as pmesh

import mfcg_oracle as orc

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

NUMBERING_CASES = [
    ((2, 2, 2), 1), ((2, 1, 1), 1), ((3, 4, 2), 2), ((2, 2, 2), 3), ((5, 3, 6), 5),
    ((8, 8, 8), 4), ((4, 4, 4), 5), ((6, 6, 6), 1), ((7, 6, 5), 4),
]

CURVED_CASES = [((3, 3, 3), 3, 4, 0.1), ((4, 3, 5), 5, 6, 0.1), ((2, 2, 2), 2, 4, 0.05)]

# 3-component Laplace (BP4 type): cells, p, nq, numbering, deformation, geometry variant
VECTOR_CASES = [((3, 2, 2), 2, 3, "default", 0.0, "affine"),
                ((4, 4, 4), 5, 6, "optimized", 0.0, "affine"),
                ((3, 3, 3), 3, 4, "default", 0.1, "final_tensor_load"),
                ((5, 4, 3), 4, 5, "default", 0.0, "affine")]


def host_tables(cells, p, *, constrain=True, numbering="default", traversal="morton", batch=None,
                deform=0.0, components=1):
    m = pmesh.build_cartesian_mesh(cells)
    if deform:
        m = pmesh.deform_mesh(m, deform)
    h = dofs.distribute_dofs(m, p, components, constrain_boundary=constrain)
    plan = dofs.make_batches(m, batch or dofs.batch_size(p, components, 8), traversal)
    if numbering == "optimized":
        h = dofs.renumber_optimized(h, plan)
    return m, h, plan


def oracle_problem(m, h, p, nq, geometry="affine", quadrature="gauss"):
    return orc.Problem(tuple(m.cells_per_dim), tuple(m.extents), m.deformation, p, nq,
                       h.cell_index_blocks, h.constrained_dofs, h.n_dofs, geometry, quadrature,
                       h.components)


def gpu_operator(m, h, plan, p, nq, variant="affine", precision="fp64", brick=(0, 0, 0),
                 quadrature="gauss"):
    from paper_2205_08909_b200.operator import MatrixFreeOperator, OperatorSpec
    spec = OperatorSpec("laplace", h.components, p, nq, pmesh.GeometryVariant(variant), quadrature)
    return MatrixFreeOperator(spec, m, h, plan, precision=precision, brick=brick)


def seeded_rhs(h, seed=0):
    """uniform[-1,1] in DEFAULT numbering, moved to the handler's numbering,
    constrained entries zeroed."""
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, h.n_dofs)
    if h.permutation is not None:
        bo = np.empty_like(b)
        bo[h.permutation] = b
        b = bo
    b[h.constrained_dofs] = 0.0
    return b


def hist_array(history):
    return np.array([[e["alpha"], e["beta"], e["gamma"], e["residual"]] for e in history])


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
