"""B200-native implementation of the merged conjugate-gradient hot path of
arXiv 2205.08909 behind the reference package's (``mfcg``) entry points:
matrix-free Laplace apply, Jacobi diagonal, CG / merged CG solve, DoF
renumbering.  See DESIGN.md; the C ABI is ``include/mfcg_b200.h``."""

__version__ = "0.1.0"

from . import dofs, mesh, tensor  # noqa: F401  (pure NumPy host modules)

__all__ = ["dofs", "mesh", "tensor", "operator", "solvers", "harness", "locality", "slabs", "build"]


def __getattr__(name):
    # operator / solvers bind the CUDA library; import them lazily so the host
    # modules stay usable for table construction on machines without it
    if name in ("operator", "solvers", "harness", "locality", "slabs", "build", "_lib"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
