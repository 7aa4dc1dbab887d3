"""The C-ABI library loads and exports every symbol include/mfcg_b200.h declares.
No compute calls: CPU only."""
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "mfcg_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mfcg_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_exports_header_symbols():
    from paper_2205_08909_b200 import _lib, build
    build.build_library()
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), f"{name} declared in mfcg_b200.h but not exported"
    assert set(names) == set(_lib.EXPORTS)


def test_error_mapping_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2205_08909_b200 import _lib
    with pytest.raises(RuntimeError):
        _lib.context(0)  # no CUDA device: the product path fails loudly, no CPU fallback


def test_host_validation_errors():
    """Argument checks that happen before any device work (operator.py:132-137,
    solvers.py:823-824)."""
    from paper_2205_08909_b200 import dofs, mesh as pmesh
    from paper_2205_08909_b200.operator import OperatorSpec
    from paper_2205_08909_b200.solvers import SolverConfig, solve
    with pytest.raises(ValueError):
        OperatorSpec("poisson", 1, 2, 3, pmesh.GeometryVariant.AFFINE)
    with pytest.raises(ValueError):
        OperatorSpec("laplace", 1, 3, 3, pmesh.GeometryVariant.AFFINE)
    with pytest.raises(ValueError):
        OperatorSpec("laplace", 1, 3, 5, pmesh.GeometryVariant.AFFINE, "gauss_lobatto")
    with pytest.raises(ValueError):
        SolverConfig(tolerance=0.0)
    with pytest.raises(ValueError):
        SolverConfig(max_iterations=0)
    with pytest.raises(ValueError):
        solve("bogus", None, None)
    with pytest.raises(ValueError):
        solve("pcg", None, None)
