"""1D quadrature rules and Lagrange tables for the B200 cell kernels (host side).

These tables are setup data: built once in Python, handed to the C-ABI
(`mfcg_op_create`) and uploaded to GPU constant memory; the hot path never
touches Python again.  Layout convention (same as the reference,
``pkg/src/mfcg/tensor.py:1-9``): cell tensors are indexed ``[z, y, x]`` with x
fastest; direction 0 is x; the reference cell is [0,1]^3.

Reference interface mirrored here (names and argument meaning):
  * ``gauss_quadrature`` / ``gauss_lobatto_quadrature``  (tensor.py:84-131)
  * ``lagrange_basis`` -> ``TensorBasis1D``               (tensor.py:223-239)
  * ``apply_1d`` / ``evaluate_*`` / ``integrate_*``       (tensor.py:242-370)
    kept as small NumPy helpers for *setup* work (host geometry tables);
    the solver never calls them -- the CUDA kernels own the sweeps.

Tables only the GPU kernels use (``collocation_gradient``, ``mass_1d``,
``stiffness_1d``) are derived from the same S, D, w.

The rules are computed with a formulation of our own (derivative recurrence
``P'_{k+1} = P'_{k-1} + (2k+1) P_k``, barycentric Lagrange weights); values
agree with the reference to a few ulp, which is all the floating-point parity
gates need (tests compare at 1e-15).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "QuadratureRule1D",
    "TensorBasis1D",
    "CellTensor",
    "gauss_quadrature",
    "gauss_lobatto_quadrature",
    "lagrange_values_1d",
    "lagrange_gradients_1d",
    "lagrange_basis",
    "apply_1d",
    "evaluate_values",
    "evaluate_gradients",
    "integrate_values",
    "integrate_gradients",
]

CellTensor = np.ndarray


@dataclass(frozen=True)
class QuadratureRule1D:
    """Points (strictly increasing, inside [0,1]) and positive weights."""

    points: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        x = np.array(self.points, dtype=np.float64)
        w = np.array(self.weights, dtype=np.float64)
        if x.ndim != 1 or x.shape != w.shape:
            raise ValueError("points and weights must be 1D arrays of equal length")
        if x.size > 1 and not np.all(x[1:] > x[:-1]):
            raise ValueError("quadrature points must be strictly increasing")
        if x.size and (x[0] < -1e-14 or x[-1] > 1.0 + 1e-14):
            raise ValueError("quadrature points must lie in [0,1]")
        if not np.all(w > 0):
            raise ValueError("quadrature weights must be positive")
        object.__setattr__(self, "points", x)
        object.__setattr__(self, "weights", w)

    def __len__(self) -> int:
        return int(self.points.size)


def _legendre_triple(n: int, t: np.ndarray):
    """(P_n, P_n', P_n'') at t in [-1,1].

    Values by Bonnet's recurrence, first and second derivatives by the
    end-point-safe recurrences  P'_{k+1} = P'_{k-1} + (2k+1) P_k  and
    P''_{k+1} = P''_{k-1} + (2k+1) P'_k."""
    t = np.asarray(t, dtype=np.float64)
    val = [np.ones_like(t), t.copy()]
    d1 = [np.zeros_like(t), np.ones_like(t)]
    d2 = [np.zeros_like(t), np.zeros_like(t)]
    for k in range(1, n):
        val.append(((2 * k + 1) * t * val[k] - k * val[k - 1]) / (k + 1))
        d1.append(d1[k - 1] + (2 * k + 1) * val[k])
        d2.append(d2[k - 1] + (2 * k + 1) * d1[k])
    return val[n], d1[n], d2[n]


def _newton(func, t, tol=1e-15, max_steps=100):
    for _ in range(max_steps):
        f, df = func(t)
        step = f / df
        t = t - step
        if np.max(np.abs(step)) < tol:
            break
    return t


def gauss_quadrature(n: int) -> QuadratureRule1D:
    """n-point Gauss-Legendre rule on [0,1], exact to degree 2n-1
    (reference: tensor.py:84-105 -- Newton on P_n from Chebyshev guesses to a
    step below 1e-15; weights 2/((1-t^2) P_n'(t)^2) mapped to [0,1])."""
    if n < 1:
        raise ValueError("gauss_quadrature requires n >= 1")
    if n == 1:
        return QuadratureRule1D(np.array([0.5]), np.array([1.0]))
    guess = -np.cos(np.pi * (np.arange(n) + 0.75) / (n + 0.5))
    t = np.sort(_newton(lambda s: _legendre_triple(n, s)[:2], guess))
    # exploit the point symmetry of the rule to remove last-ulp asymmetry
    t = 0.5 * (t - t[::-1])
    _, dp, _ = _legendre_triple(n, t)
    w = 2.0 / ((1.0 - t * t) * dp * dp)
    return QuadratureRule1D(0.5 * (t + 1.0), 0.5 * w)


def gauss_lobatto_quadrature(n: int) -> QuadratureRule1D:
    """n-point Gauss-Lobatto rule on [0,1] with both end points, exact to
    degree 2n-3 (reference: tensor.py:108-131).  Interior nodes are the roots
    of P'_{n-1}; weights 2/(m(m+1) P_m(t)^2), m = n-1."""
    if n < 2:
        raise ValueError("gauss_lobatto_quadrature requires n >= 2")
    m = n - 1
    if n == 2:
        t = np.array([-1.0, 1.0])
    else:
        guess = -np.cos(np.pi * np.arange(1, m) / m)
        inner = np.sort(_newton(lambda s: _legendre_triple(m, s)[1:], guess))
        inner = 0.5 * (inner - inner[::-1])
        t = np.concatenate(([-1.0], inner, [1.0]))
    pm, _, _ = _legendre_triple(m, t)
    w = 2.0 / (m * (m + 1) * pm * pm)
    return QuadratureRule1D(0.5 * (t + 1.0), 0.5 * w)


def _bary_weights(nodes: np.ndarray) -> np.ndarray:
    diff = nodes[:, None] - nodes[None, :]
    np.fill_diagonal(diff, 1.0)
    return 1.0 / np.prod(diff, axis=1)


def lagrange_values_1d(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """V[q, i] = l_i(x_q) for the Lagrange polynomials through `nodes`
    (reference tensor.py:134-145), evaluated in product form with barycentric
    denominators so that coinciding points give exact 0/1 entries."""
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    n = nodes.size
    wb = _bary_weights(nodes)
    gap = x[:, None] - nodes[None, :]            # (q, j)
    V = np.empty((x.size, n))
    for i in range(n):
        V[:, i] = wb[i] * np.prod(np.delete(gap, i, axis=1), axis=1)
    return V


def lagrange_gradients_1d(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """G[q, i] = l_i'(x_q) (reference tensor.py:148-164): product rule over the
    omitted factor, valid also where x_q coincides with a node."""
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    n = nodes.size
    wb = _bary_weights(nodes)
    gap = x[:, None] - nodes[None, :]
    G = np.zeros((x.size, n))
    for i in range(n):
        others = [j for j in range(n) if j != i]
        acc = np.zeros(x.size)
        for m in others:
            keep = [j for j in others if j != m]
            acc += np.prod(gap[:, keep], axis=1) if keep else 1.0
        G[:, i] = wb[i] * acc
    return G


@dataclass(frozen=True)
class TensorBasis1D:
    """Degree-p Lagrange basis on Gauss-Lobatto nodes tabulated at a quadrature
    rule: ``shape_values[q,i] = phi_i(x_q)``, ``shape_gradients[q,i] = phi_i'(x_q)``
    (reference tensor.py:200-221)."""

    degree: int
    node_points: np.ndarray
    quadrature: QuadratureRule1D
    shape_values: np.ndarray
    shape_gradients: np.ndarray

    @property
    def n_q(self) -> int:
        return len(self.quadrature)

    @property
    def collocation_gradient(self) -> np.ndarray:
        """Dc[q, r] = derivative at x_q of the Lagrange polynomial through the
        quadrature points that is 1 at x_r.  With n_q >= p+1 the interpolant
        through the quadrature points reproduces the degree-p field, so
        ``Dc @ shape_values == shape_gradients`` up to rounding; the general-
        geometry GPU kernel uses it to get all three gradient components from
        ONE interpolated field (3 + 3 sweeps instead of 9)."""
        pts = self.quadrature.points
        return lagrange_gradients_1d(pts, pts)

    @property
    def mass_1d(self) -> np.ndarray:
        """M[i, j] = sum_q w_q phi_i(x_q) phi_j(x_q) on [0,1]."""
        w = self.quadrature.weights
        return self.shape_values.T @ (w[:, None] * self.shape_values)

    @property
    def stiffness_1d(self) -> np.ndarray:
        """K[i, j] = sum_q w_q phi_i'(x_q) phi_j'(x_q) on [0,1]."""
        w = self.quadrature.weights
        return self.shape_gradients.T @ (w[:, None] * self.shape_gradients)


def lagrange_basis(p: int, quad: QuadratureRule1D) -> TensorBasis1D:
    """Degree-p basis (Gauss-Lobatto support) tabulated at `quad`."""
    if p < 1:
        raise ValueError("polynomial degree must be >= 1")
    nodes = gauss_lobatto_quadrature(p + 1).points
    return TensorBasis1D(
        degree=p,
        node_points=nodes,
        quadrature=quad,
        shape_values=lagrange_values_1d(nodes, quad.points),
        shape_gradients=lagrange_gradients_1d(nodes, quad.points),
    )


# ---------------------------------------------------------------------------
# setup-time NumPy sweeps (not on the solver path)


def apply_1d(matrix: np.ndarray, tensor: np.ndarray, direction: int,
             transpose: bool = False) -> np.ndarray:
    """Contract `matrix` (or its transpose) along one direction of a cell
    tensor (0 = x = last axis); leading batch axes pass through."""
    if direction not in (0, 1, 2):
        raise ValueError("direction must be 0, 1 or 2")
    mat = matrix.T if transpose else matrix
    axis = tensor.ndim - 1 - direction
    if tensor.shape[axis] != mat.shape[1]:
        raise ValueError(
            f"tensor extent {tensor.shape[axis]} in direction {direction} "
            f"does not match matrix columns {mat.shape[1]}")
    out = np.tensordot(tensor, mat, axes=([axis], [1]))
    return np.moveaxis(out, -1, axis)


def _tensor_sweep(basis: TensorBasis1D, tensor, grad_dir, transpose):
    out = tensor
    for d in range(3):
        mat = basis.shape_gradients if d == grad_dir else basis.shape_values
        out = apply_1d(mat, out, d, transpose)
    return out


def evaluate_values(basis: TensorBasis1D, cell_dofs: np.ndarray) -> np.ndarray:
    """Nodal coefficients -> values at the quadrature points."""
    return _tensor_sweep(basis, cell_dofs, None, False)


def evaluate_gradients(basis: TensorBasis1D, cell_dofs: np.ndarray) -> np.ndarray:
    """Reference-space gradient at all quadrature points; the three derivative
    components are stacked on a new leading axis."""
    return np.stack([_tensor_sweep(basis, cell_dofs, c, False) for c in range(3)])


def integrate_values(basis: TensorBasis1D, quad_data: np.ndarray) -> np.ndarray:
    """Adjoint of :func:`evaluate_values`."""
    return _tensor_sweep(basis, quad_data, None, True)


def integrate_gradients(basis: TensorBasis1D, quad_data: np.ndarray) -> np.ndarray:
    """Adjoint of :func:`evaluate_gradients` (components on axis 0)."""
    if quad_data.shape[0] != 3:
        raise ValueError("quad_data must stack 3 gradient components on axis 0")
    return sum(_tensor_sweep(basis, quad_data[c], c, True) for c in range(3))
