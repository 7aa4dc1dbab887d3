"""Small merged solve + apply for compute-sanitizer runs (memcheck / racecheck), partial bricks included."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
import numpy as np
from paper_2205_08909_b200 import dofs, mesh as pmesh
from paper_2205_08909_b200.operator import MatrixFreeOperator, OperatorSpec
from paper_2205_08909_b200.solvers import SolverConfig, solve

for cells, p, variant, deform in [((5, 3, 3), 5, "affine", 0.0), ((3, 4, 2), 3, "final_tensor_load", 0.05)]:
    m = pmesh.build_cartesian_mesh(cells)
    if deform:
        m = pmesh.deform_mesh(m, deform)
    h = dofs.distribute_dofs(m, p, 1, constrain_boundary=True)
    plan = dofs.make_batches(m, 8, "morton")
    op = MatrixFreeOperator(OperatorSpec("laplace", 1, p, p + 1, pmesh.GeometryVariant(variant)), m, h, plan,
                            brick=(0, 0, 2))
    b = np.random.default_rng(0).uniform(-1, 1, h.n_dofs)
    b[h.constrained_dofs] = 0
    op.apply(b)
    res = solve("combined_pcg", op, b, minv=op.compute_diagonal(), config=SolverConfig(fixed_iterations=4))
    res2 = solve("pcg", op, b, minv=op.compute_diagonal(), config=SolverConfig(fixed_iterations=4))
    print(cells, p, variant, res.residual, res2.residual)
