"""GPU parity: every call goes through the C ABI (libmfcg_b200.so) and is checked
against the CPU oracle on the same seeded inputs and against the committed
reference fixtures.  Tolerances: integer tables bit-exact; one apply / diagonal
1e-12 relative; CG scalars 1e-10 while the reference's own re-ordering envelope
allows it."""
import numpy as np
import pytest

import mfcg_oracle as orc
from _problems import (APPLY_CASES, gpu_operator, hist_array, host_tables, oracle_problem, rel,
                       seeded_rhs)

pytestmark = pytest.mark.gpu


def _solvers():
    from paper_2205_08909_b200 import solvers
    return solvers


@pytest.mark.parametrize("ci", range(len(APPLY_CASES)))
def test_apply_diag_perm_vs_fixture(golden, ci):
    cells, p, nq, numb, con = APPLY_CASES[ci]
    g = golden["apply"]
    m, h, plan = host_tables(cells, p, constrain=con, numbering=numb)
    op = gpu_operator(m, h, plan, p, nq)
    perm = op.device_permutation()
    assert np.array_equal(np.sort(perm), np.arange(h.n_dofs)), "brick numbering is not a bijection"
    u = g[f"c{ci}_u"]
    Au = op.apply(u)
    assert rel(Au, g[f"c{ci}_Au"]) < 1e-12
    if con:
        assert np.array_equal(Au[h.constrained_dofs], u[h.constrained_dofs])
        assert rel(op.compute_diagonal().inverse_diagonal, g[f"c{ci}_invdiag"]) < 1e-12
    out = np.empty_like(u)
    assert op.apply(u, out=out) is out and np.array_equal(out, Au) or rel(out, Au) < 1e-14
    with pytest.raises(ValueError):
        op.apply(u[:-1])


@pytest.mark.parametrize("brick", [(1, 1, 1), (2, 3, 2), (3, 3, 1), (3, 2, 5)])
def test_apply_independent_of_brick_shape(brick):
    cells, p, nq = (7, 5, 6), 5, 6
    m, h, plan = host_tables(cells, p)
    prob = oracle_problem(m, h, p, nq)
    u = np.random.default_rng(5).standard_normal(h.n_dofs)
    ref = orc.apply(prob, u)
    op = gpu_operator(m, h, plan, p, nq, brick=brick)
    assert op.info()["brick"] == brick
    assert rel(op.apply(u), ref) < 1e-12
    assert rel(op.compute_diagonal().inverse_diagonal, orc.inverse_diagonal(prob)) < 1e-12


def test_linearity_symmetry_nullspace():
    m, h, plan = host_tables((6, 5, 9), 5, constrain=False)
    op = gpu_operator(m, h, plan, 5, 6)
    rng = np.random.default_rng(11)
    a, b = rng.standard_normal(h.n_dofs), rng.standard_normal(h.n_dofs)
    Aa, Ab = op.apply(a), op.apply(b)
    assert rel(op.apply(2.0 * a - 3.0 * b), 2.0 * Aa - 3.0 * Ab) < 1e-12
    assert abs(a @ Ab - b @ Aa) < 1e-10 * abs(a @ Ab)
    assert np.max(np.abs(op.apply(np.ones(h.n_dofs)))) < 1e-11


def test_config1_solves_vs_reference(golden):
    """BASELINE configs[0]: 8^3 cells Q4, 100 fixed iterations, all four variants."""
    S = _solvers()
    g = golden["config1"]
    m, h, plan = host_tables((8, 8, 8), 4)
    op = gpu_operator(m, h, plan, 4, 5)
    b = g["b"]
    assert np.array_equal(b, seeded_rhs(h))
    assert rel(op.apply(b), g["Ab"]) < 1e-12
    minv = op.compute_diagonal()
    assert rel(minv.inverse_diagonal, g["invdiag"]) < 1e-12
    cfg = S.SolverConfig(fixed_iterations=100)
    for variant in ("pcg", "combined_pcg", "cg", "combined_cg"):
        for fused in ((True, False) if variant.startswith("combined") else (True,)):
            res = S.solve(variant, op, b, minv=minv, config=S.SolverConfig(fixed_iterations=100, fused=fused))
            H, R = hist_array(res.history), g[f"{variant}_hist"]
            assert res.iterations == 100 and res.matvecs == 100 and H.shape == R.shape
            dev = np.abs(H[:, 3] - R[:, 3]) / R[:, 3]
            xdev = rel(res.x, g[f"{variant}_x"])
            if variant in ("pcg", "combined_pcg"):
                E = g[f"{variant}_hist_reordered"]
                env = np.maximum.accumulate(np.abs(E[:, 3] - R[:, 3]) / R[:, 3])
                strict = env < 1e-11
                assert dev[strict].max() < 1e-10, (variant, fused, dev[strict].max())
                # beyond that point CG amplifies rounding noise exponentially and the GPU's
                # atomic accumulation order changes from run to run: stay within one order
                # of magnitude of the reference's own re-ordering envelope (SURVEY.md 8c iii).
                # Observed over repeated runs on B200: combined_pcg 0.2 .. 0.5 x the envelope, pcg
                # 2 .. 11 x (its envelope is the smaller one: 2e-8 at iteration 100 vs 3e-7), so the
                # gate is 10 x for the merged variant and 3 x the observed maximum for pcg.
                ratio = float(np.max(dev[~strict] / (env[~strict] + 1e-11)))
                print(f"config1 {variant} fused={fused}: strict zone {int(strict.sum())} its, max dev there "
                      f"{dev[strict].max():.2e}; beyond: max dev/envelope {ratio:.2f}; |x - x_ref|/|x_ref| {xdev:.2e}")
                factor = 10 if variant == "combined_pcg" else 30
                assert np.all(dev[~strict] <= factor * env[~strict] + 1e-10), (variant, fused, ratio)
            else:
                print(f"config1 {variant}: max residual dev over 100 its {dev.max():.2e}; x dev {xdev:.2e}")
            assert dev[:40].max() < 1e-10
            for col in range(3):
                assert rel(H[:40, col], R[:40, col]) < 1e-10, (variant, fused, col)
            # observed on B200: 6e-11 .. 2e-9 (the reference against a re-ordered copy of itself: 6e-11 .. 3e-9)
            assert xdev < 1e-8, (variant, fused, xdev)
            # true residual of the returned iterate agrees with the recurred one
            true_res = np.linalg.norm(b - op.apply(res.x)) / np.linalg.norm(b)
            assert abs(true_res - res.residual) < 1e-9
    # a preconditioner passed as a plain array gives the same history
    res2 = S.solve("combined_pcg", op, b, minv=np.array(minv.inverse_diagonal), config=cfg)
    res1 = S.solve("combined_pcg", op, b, minv=minv, config=cfg)
    assert rel(hist_array(res2.history)[:40], hist_array(res1.history)[:40]) < 1e-10


def test_tolerance_termination_and_edge_cases(golden):
    S = _solvers()
    g = golden["config1"]
    m, h, plan = host_tables((8, 8, 8), 4)
    op = gpu_operator(m, h, plan, 4, 5)
    minv = op.compute_diagonal()
    for variant in ("pcg", "combined_pcg"):
        res = S.solve(variant, op, g["b"], minv=minv, config=S.SolverConfig(tolerance=1e-6, max_iterations=500))
        assert [res.iterations, int(res.converged)] == list(g[f"{variant}_tol_iters"])
        assert len(res.history) == res.iterations
        assert res.matvecs == res.iterations   # solvers.py:218, 705 (launches behind the converged iteration are no-ops)
        assert rel(hist_array(res.history)[:, 3], g[f"{variant}_tol_hist"][:, 3]) < 1e-8
    zero = S.solve("combined_pcg", op, np.zeros(h.n_dofs), minv=minv)
    assert zero.iterations == 0 and zero.converged and not zero.history and np.all(zero.x == 0)
    with pytest.raises(ValueError):
        S.solve("pcg", op, g["b"])
    with pytest.raises(ValueError):
        S.solve("combined_pcg", op, g["b"][:-1], minv=minv)
    with pytest.raises(ValueError):
        S.solve("pcg", op, g["b"], minv=np.ones(5))
    # merged vs standard alpha/beta over 10 iterations (reference tests/test_solvers.py:115-131)
    a = hist_array(S.solve("pcg", op, g["b"], minv=minv, config=S.SolverConfig(fixed_iterations=10)).history)
    c = hist_array(S.solve("combined_pcg", op, g["b"], minv=minv, config=S.SolverConfig(fixed_iterations=10)).history)
    assert rel(a[:, 0], c[:, 0]) < 1e-8 and rel(a[:, 1], c[:, 1]) < 1e-8
    # force_x_updates gives the same solution (tests/test_solvers.py:252-257)
    x1 = S.solve("combined_pcg", op, g["b"], minv=minv, config=S.SolverConfig(fixed_iterations=31)).x
    x2 = S.solve("combined_pcg", op, g["b"], minv=minv,
                 config=S.SolverConfig(fixed_iterations=31, force_x_updates=True)).x
    assert rel(x1, x2) < 1e-9
    # breakdown: negative "preconditioner" (tests/test_solvers.py:185-227)
    with pytest.raises(S.SolverBreakdown):
        S.solve("combined_pcg", op, g["b"], minv=-np.ones(h.n_dofs))


def test_q5_small_vs_reference(golden):
    """BASELINE configs[1], rungs 4^3 and 6^3 (Q5, 200 iterations), default and optimized numbering."""
    S = _solvers()
    g = golden["q5_small"]
    for n, numb in ((4, "default"), (6, "default"), (4, "optimized")):
        tag = f"n{n}_{numb}"
        m, h, plan = host_tables((n, n, n), 5, numbering=numb)
        op = gpu_operator(m, h, plan, 5, 6)
        b = g[f"{tag}_b"]
        assert np.array_equal(b, seeded_rhs(h))
        minv = op.compute_diagonal()
        for variant in ("pcg", "combined_pcg"):
            res = S.solve(variant, op, b, minv=minv, config=S.SolverConfig(fixed_iterations=200))
            H, R = hist_array(res.history), g[f"{tag}_{variant}_hist"]
            assert H.shape == R.shape
            assert (np.abs(H[:40, 3] - R[:40, 3]) / R[:40, 3]).max() < 1e-10, (tag, variant)
            assert rel(H[:40, :2], R[:40, :2]) < 1e-10


def test_midsize_vs_oracle_and_roundtrip():
    """16^3 cells Q5 (5.3e5 DoFs): apply vs oracle, solve to tolerance, true residual."""
    S = _solvers()
    m, h, plan = host_tables((16, 16, 16), 5, numbering="optimized")
    prob = oracle_problem(m, h, 5, 6)
    op = gpu_operator(m, h, plan, 5, 6)
    u = np.random.default_rng(2).standard_normal(h.n_dofs)
    assert rel(op.apply(u), orc.apply(prob, u)) < 1e-12
    minv = op.compute_diagonal()
    assert rel(minv.inverse_diagonal, orc.inverse_diagonal(prob)) < 1e-12
    b = seeded_rhs(h)
    res = S.solve("combined_pcg", op, b, minv=minv, config=S.SolverConfig(tolerance=1e-9, max_iterations=2000))
    assert res.converged
    assert np.linalg.norm(b - op.apply(res.x)) / np.linalg.norm(b) < 2e-9
    ref = S.solve("pcg", op, b, minv=minv, config=S.SolverConfig(tolerance=1e-9, max_iterations=2000))
    assert ref.converged and abs(ref.iterations - res.iterations) <= 2
    assert rel(res.x, ref.x) < 1e-6


def test_fp32_variant():
    """fp32 vectors/operator (BASELINE configs[3]): 1e-4 relative against the fp64 oracle."""
    S = _solvers()
    m, h, plan = host_tables((6, 6, 6), 3)
    prob = oracle_problem(m, h, 3, 4)
    op = gpu_operator(m, h, plan, 3, 4, precision="fp32")
    u = np.random.default_rng(4).standard_normal(h.n_dofs)
    assert rel(op.apply(u), orc.apply(prob, u)) < 1e-5
    minv = orc.inverse_diagonal(prob)
    b = seeded_rhs(h)
    x, k, r, conv, hist = orc.combined_pcg(lambda v: orc.apply(prob, v), b, minv, fixed_iterations=20)
    res = S.solve("combined_pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=20))
    assert rel(hist_array(res.history)[:, 3], hist_array(hist)[:, 3]) < 1e-4
    assert rel(res.x, x) < 1e-4


@pytest.mark.parametrize("p", range(1, 9))
def test_fp32_all_degrees(p):
    """BASELINE configs[3]: every degree in fp32 (vectors and operator), 1e-4 relative against the fp64 oracle:
    one apply, the 20-iteration merged-PCG residual history and the iterate."""
    S = _solvers()
    cells = {1: (19, 18, 5), 2: (11, 12, 4), 3: (7, 8, 3), 4: (6, 5, 3), 5: (5, 4, 3), 6: (4, 3, 3),
             7: (3, 3, 3), 8: (3, 2, 3)}[p]
    m, h, plan = host_tables(cells, p)
    prob = oracle_problem(m, h, p, p + 1)
    op = gpu_operator(m, h, plan, p, p + 1, precision="fp32")
    u = np.random.default_rng(40 + p).standard_normal(h.n_dofs)
    assert rel(op.apply(u), orc.apply(prob, u)) < 1e-5
    minv = orc.inverse_diagonal(prob)
    b = seeded_rhs(h)
    for variant, fn in (("combined_pcg", orc.combined_pcg), ("pcg", orc.pcg)):
        x, k, r, conv, hist = fn(lambda v: orc.apply(prob, v), b, minv, fixed_iterations=20)
        res = S.solve(variant, op, b, minv=minv, config=S.SolverConfig(fixed_iterations=20))
        assert rel(hist_array(res.history)[:, 3], hist_array(hist)[:, 3]) < 1e-4, (p, variant)
        assert rel(res.x, x) < 1e-4, (p, variant)
    # the library's own diagonal (computed in fp64, applied in fp32) gives the same history
    res2 = S.solve("combined_pcg", op, b, minv=op.compute_diagonal(), config=S.SolverConfig(fixed_iterations=20))
    x, k, r, conv, hist = orc.combined_pcg(lambda v: orc.apply(prob, v), b, minv, fixed_iterations=20)
    assert rel(hist_array(res2.history)[:, 3], hist_array(hist)[:, 3]) < 1e-4


@pytest.mark.parametrize("p", range(1, 9))
def test_all_degrees_apply_and_short_solve(p):
    S = _solvers()
    cells = {1: (19, 18, 5), 2: (11, 12, 4), 3: (7, 8, 3), 4: (6, 5, 3), 5: (5, 4, 3), 6: (4, 3, 3),
             7: (3, 3, 3), 8: (3, 2, 3)}[p]
    m, h, plan = host_tables(cells, p)
    prob = oracle_problem(m, h, p, p + 1)
    op = gpu_operator(m, h, plan, p, p + 1)
    u = np.random.default_rng(p).standard_normal(h.n_dofs)
    assert rel(op.apply(u), orc.apply(prob, u)) < 1e-12
    minv_ref = orc.inverse_diagonal(prob)
    minv = op.compute_diagonal()
    assert rel(minv.inverse_diagonal, minv_ref) < 1e-12
    b = seeded_rhs(h)
    mv = lambda v: orc.apply(prob, v)
    for variant, fn in (("pcg", orc.pcg), ("combined_pcg", orc.combined_pcg)):
        x, k, r, conv, hist = fn(mv, b, minv_ref, fixed_iterations=15)
        res = S.solve(variant, op, b, minv=minv, config=S.SolverConfig(fixed_iterations=15))
        assert rel(hist_array(res.history), hist_array(hist)) < 1e-10, (p, variant)
        assert rel(res.x, x) < 1e-10


# ---------------------------------------------------------------------------
# curved meshes (BASELINE configs[2]): tri-quadratic geometry, stored and on-the-fly variants

from _problems import CURVED_CASES  # noqa: E402


@pytest.mark.parametrize("ci", [0, 1])
def test_curved_variants_vs_reference(golden, ci):
    S = _solvers()
    cells, p, nq, amp = CURVED_CASES[ci]
    g = golden["curved"]
    m, h, plan = host_tables(cells, p, deform=amp)
    u = g[f"k{ci}_u"]
    ops = {}
    for variant in ("final_tensor_load", "inverse_jacobian_load", "quadratic_compute"):
        op = ops[variant] = gpu_operator(m, h, plan, p, nq, variant=variant)
        # all variants describe the same map (reference tests/test_operator.py:82-88)
        assert rel(op.apply(u), g[f"k{ci}_Au"]) < 1e-12, variant
        assert rel(op.compute_diagonal().inverse_diagonal, g[f"k{ci}_invdiag"]) < 1e-12, variant
    geo = ops["final_tensor_load"].device_geometry()
    assert rel(geo["final_tensor"], g[f"k{ci}_final_tensor"]) < 1e-12
    geo = ops["inverse_jacobian_load"].device_geometry()
    assert rel(geo["inverse_jacobian"], g[f"k{ci}_inverse_jacobian"]) < 1e-12
    assert rel(geo["jxw"], g[f"k{ci}_jxw"]) < 1e-12
    b = g[f"k{ci}_b"]
    R = g[f"k{ci}_combined_pcg_hist"]
    for variant, op in ops.items():
        res = S.solve("combined_pcg", op, b, minv=op.compute_diagonal(), config=S.SolverConfig(fixed_iterations=40))
        H = hist_array(res.history)
        assert (np.abs(H[:30, 3] - R[:30, 3]) / R[:30, 3]).max() < 1e-10, variant
        assert rel(H[:30, :2], R[:30, :2]) < 1e-10, variant
        assert rel(res.x, g[f"k{ci}_combined_pcg_x"]) < 1e-8, variant
        ref = S.solve("pcg", op, b, minv=op.compute_diagonal(), config=S.SolverConfig(fixed_iterations=40))
        assert rel(hist_array(ref.history)[:30, 3], R[:30, 3]) < 1e-8


def test_curved_midsize_vs_oracle_and_errors():
    cells, p, nq, amp = (9, 7, 6), 5, 6, 0.1
    m, h, plan = host_tables(cells, p, deform=amp)
    prob = oracle_problem(m, h, p, nq, geometry="curved")
    u = np.random.default_rng(8).standard_normal(h.n_dofs)
    ref = orc.apply(prob, u)
    for variant in ("final_tensor_load", "quadratic_compute"):
        op = gpu_operator(m, h, plan, p, nq, variant=variant)
        assert rel(op.apply(u), ref) < 1e-12
    assert op.info()["geometry_bytes"] > 0
    with pytest.raises(ValueError):            # affine on a deformed mesh (mesh.py:214-216)
        gpu_operator(m, h, plan, p, nq, variant="affine")
    # n_q > p+1 on curved meshes (operator.py:69-70; BP3 / BP4 use p+2): the cell-by-cell path, every variant
    for nq2 in (nq + 1, nq + 3):
        prob2 = oracle_problem(m, h, p, nq2, geometry="curved")
        ref2 = orc.apply(prob2, u)
        for variant in ("final_tensor_load", "inverse_jacobian_load", "quadratic_compute"):
            assert rel(gpu_operator(m, h, plan, p, nq2, variant=variant).apply(u), ref2) < 1e-12, (nq2, variant)
    # undeformed mesh: final-tensor variant == affine (reference tests/test_operator.py:90-95)
    m0, h0, plan0 = host_tables((5, 4, 3), 3)
    u0 = np.random.default_rng(9).standard_normal(h0.n_dofs)
    a = gpu_operator(m0, h0, plan0, 3, 4).apply(u0)
    f = gpu_operator(m0, h0, plan0, 3, 4, variant="final_tensor_load").apply(u0)
    assert rel(f, a) < 1e-12


# ---------------------------------------------------------------------------
# 3 components (SURVEY.md 8f row 3, BP4 type): the scalar operator on every component

from _problems import VECTOR_CASES  # noqa: E402


@pytest.mark.parametrize("ci", range(len(VECTOR_CASES)))
def test_three_components_vs_reference(golden, ci):
    S = _solvers()
    cells, p, nq, numbering, amp, variant = VECTOR_CASES[ci]
    g = golden["vector3"]
    m, h, plan = host_tables(cells, p, numbering=numbering, deform=amp, components=3)
    op = gpu_operator(m, h, plan, p, nq, variant=variant)
    assert op.components == 3 and op.n_dofs == h.n_dofs == op.info()["n_dofs"]
    u = g[f"v{ci}_u"]
    Au = op.apply(u)
    assert rel(Au, g[f"v{ci}_Au"]) < 1e-12
    assert np.array_equal(Au[h.constrained_dofs], u[h.constrained_dofs])      # operator.py:359-360
    minv = op.compute_diagonal()
    assert minv.inverse_diagonal.shape == (h.n_dofs // 3,)                    # operator.py:90
    assert rel(minv.inverse_diagonal, g[f"v{ci}_invdiag"]) < 1e-12
    b = g[f"v{ci}_b"]
    for name in ("pcg", "combined_pcg", "combined_cg"):
        R = g[f"v{ci}_{name}_hist"]
        for mv in ((minv, minv.inverse_diagonal.copy()) if name != "combined_cg" else (None,)):
            # the operator's own diagonal (device copy / on-the-fly) and a caller-supplied array
            res = S.solve(name, op, b, minv=mv, config=S.SolverConfig(fixed_iterations=30))
            H = hist_array(res.history)
            assert res.iterations == 30 and res.matvecs == 30
            # strict while the residual is far from the rounding floor of these tiny systems
            # (CG amplifies summation-order noise once it is not)
            k = np.flatnonzero(R[:20, 3] > 1e-6)
            assert len(k) >= 8
            assert (np.abs(H[k, 3] - R[k, 3]) / R[k, 3]).max() < 1e-10, name
            assert rel(H[k, :2], R[k, :2]) < 1e-10, name
            assert rel(res.x, g[f"v{ci}_{name}_x"]) < 1e-8, name
    unf = S.solve("combined_pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=30, fused=False))
    R = g[f"v{ci}_combined_pcg_hist"]
    k = np.flatnonzero(R[:20, 3] > 1e-6)
    assert rel(hist_array(unf.history)[k, 3], R[k, 3]) < 1e-10
    with pytest.raises(ValueError):            # one diagonal value per NODE (solvers.py:617-619)
        S.solve("combined_pcg", op, b, minv=np.ones(h.n_dofs))


def test_three_components_curved_one_launch(monkeypatch):
    """Stored geometry with three components: one launch, the blocks of a brick next to each other so that its
    geometry is read from HBM once (MFCG_COMP_INTERLEAVE=0: one launch per component).  Same results either way."""
    S = _solvers()
    cells, p, nq, amp = (9, 7, 6), 4, 5, 0.08
    m, h, plan = host_tables(cells, p, numbering="optimized", deform=amp, components=3)
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, h.n_dofs)
    b = rng.uniform(-1, 1, h.n_dofs)
    b[h.constrained_dofs] = 0.0
    out = {}
    variants = ("final_tensor_load", "inverse_jacobian_load")
    for flag in ("0", "1"):
        monkeypatch.setenv("MFCG_COMP_INTERLEAVE", flag)
        for variant in variants:
            op = gpu_operator(m, h, plan, p, nq, variant=variant)
            res = S.solve("combined_pcg", op, b, minv=op.compute_diagonal(), config=S.SolverConfig(fixed_iterations=25))
            std = S.solve("pcg", op, b, minv=op.compute_diagonal(), config=S.SolverConfig(fixed_iterations=25))
            out[flag, variant] = (op.apply(u), hist_array(res.history), res.x, hist_array(std.history))
    for variant in variants:
        a0, h0, x0, s0 = out["0", variant]
        a1, h1, x1, s1 = out["1", variant]
        assert rel(a1, a0) < 1e-14 and rel(h1[:, 3], h0[:, 3]) < 1e-11 and rel(x1, x0) < 1e-11
        assert rel(s1[:, 3], s0[:, 3]) < 1e-11
        # components must not mix: component c of A u is the scalar operator on component c
        assert rel(h1[:12, 3], s1[:12, 3]) < 1e-6


def test_three_components_midsize_vs_oracle():
    """Q5, ragged brick grid, three components against the CPU oracle; a vector whose components
    differ must not mix them."""
    cells, p, nq = (9, 6, 7), 5, 6
    m, h, plan = host_tables(cells, p, components=3)
    prob = oracle_problem(m, h, p, nq)
    op = gpu_operator(m, h, plan, p, nq)
    u = np.random.default_rng(12).standard_normal(h.n_dofs)
    assert rel(op.apply(u), orc.apply(prob, u)) < 1e-12
    only1 = np.zeros_like(u)
    only1[1::3] = u[1::3]
    out = op.apply(only1)
    free = np.ones(h.n_dofs, bool)
    free[h.constrained_dofs] = False
    assert not out[0::3][free[0::3]].any() and not out[2::3][free[2::3]].any()
    with pytest.raises(ValueError):            # partial-node constraints (dofs.py:329-330)
        bad = dofs_replace_constraints(h, h.constrained_dofs[1:])
        gpu_operator(m, bad, plan, p, nq)


def dofs_replace_constraints(h, constrained):
    import dataclasses
    return dataclasses.replace(h, constrained_dofs=np.asarray(constrained, dtype=np.int64))


# ---------------------------------------------------------------------------
# BASELINE sizes: no oracle can run there, so size-independent properties (the prompt's
# "encode -> decode round trips, linearity, checksums"): true vs recurred residual, merged vs
# standard scalars, linearity of the operator, constrained rows copied through bit-exactly.


@pytest.mark.parametrize("n", [73, 116])
def test_full_size_properties(n):
    """Q5 at 73^3 (4.9e7 DoFs, the >= 5e7 target size) and 116^3 (1.96e8 DoFs, top rung of configs[1])."""
    S = _solvers()
    p = 5
    m, h, plan = host_tables((n, n, n), p)
    op = gpu_operator(m, h, plan, p, p + 1)
    b = seeded_rhs(h)
    minv = op.compute_diagonal()
    iters = 30
    mer = S.solve("combined_pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=iters))
    std = S.solve("pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=iters))
    Hm, Hs = hist_array(mer.history), hist_array(std.history)
    assert rel(Hm[:, 0], Hs[:, 0]) < 1e-8 and rel(Hm[:, 1], Hs[:, 1]) < 1e-8   # alpha, beta
    assert rel(Hm[:, 3], Hs[:, 3]) < 1e-8                                       # residual history
    bn = np.linalg.norm(b)
    Ax = op.apply(mer.x)
    assert abs(np.linalg.norm(b - Ax) / bn - mer.residual) < 1e-9               # recurred == true residual
    assert np.array_equal(Ax[h.constrained_dofs], mer.x[h.constrained_dofs])    # identity rows, bit-exact
    assert rel(mer.x, std.x) < 1e-7
    # linearity: A(2x - 3b) == 2 Ax - 3 Ab
    Ab = op.apply(b)
    assert rel(op.apply(2.0 * mer.x - 3.0 * b), 2.0 * Ax - 3.0 * Ab) < 1e-12
    # energy checksum: x.b == x.A x up to the residual (symmetric positive operator)
    assert abs(mer.x @ Ax - mer.x @ b) <= 2 * mer.residual * bn * np.linalg.norm(mer.x)


def test_repeated_solves_on_ragged_brick_grid():
    """The persistent kernel walks several bricks per block and pipelines across brick boundaries; on a
    49 x 49 x 20 mesh (845 bricks of 4 x 4 x 4 cells with 1-cell-wide ragged bricks, 5-6 bricks per block)
    every block changes brick shape several times per launch.  A mis-ordered hand-over between the roles
    shows up as a history that differs between identical solves (it did: NT = 5 transient slots with four
    update warps let a warp wait two barrier phases ahead, once in a few hundred launches), so: the
    first solve against the oracle, and 40 repeated 200-iteration solves against the first."""
    S = _solvers()
    p = 5
    m, h, plan = host_tables((49, 49, 20), p)
    op = gpu_operator(m, h, plan, p, p + 1, brick=(0, 0, 4))
    assert op.info()["n_bricks"] == 845
    b = seeded_rhs(h)
    minv = op.compute_diagonal()
    prob = oracle_problem(m, h, p, p + 1)
    first = S.solve("combined_pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=12))
    import mfcg_oracle_c as oc
    if oc.available():
        cp = oc.CProblem(prob)
        _, _, hist = cp.combined_pcg(b, minv.inverse_diagonal, 12)   # hist[k] = alpha, beta, gamma, residual
        assert rel(hist_array(first.history)[:, 3], hist[:, 3]) < 1e-10
    ref = None
    worst = 0.0
    for _ in range(40):
        res = S.solve("combined_pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=200))
        H = hist_array(res.history)[:, 3]
        if ref is None:
            ref = H
        worst = max(worst, float(np.max(np.abs(H - ref) / ref)))
    print(f"repeated ragged solves: max relative history deviation {worst:.2e}")
    assert worst < 1e-9   # run-to-run differences come from the order of the RED.F64 adds only


@pytest.mark.parametrize("variant", ["final_tensor_load", "inverse_jacobian_load", "quadratic_compute"])
def test_full_size_properties_curved(variant):
    """BASELINE configs[2]: Q5 on 96^3 cells deformed by 0.1 sin sin sin (1.11e8 DoFs), each geometry variant.
    No oracle runs there; size-independent properties as in test_full_size_properties, plus agreement of the
    variants with each other through the residual history (the reference pins its variants to each other at
    1e-12 on one apply, tests/test_operator.py:82-88)."""
    S = _solvers()
    p, n = 5, 96
    m, h, plan = host_tables((n, n, n), p, deform=0.1)
    op = gpu_operator(m, h, plan, p, p + 1, variant=variant)
    b = seeded_rhs(h)
    minv = op.compute_diagonal()
    iters = 30
    mer = S.solve("combined_pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=iters))
    std = S.solve("pcg", op, b, minv=minv, config=S.SolverConfig(fixed_iterations=iters))
    Hm, Hs = hist_array(mer.history), hist_array(std.history)
    assert rel(Hm[:, 0], Hs[:, 0]) < 1e-8 and rel(Hm[:, 1], Hs[:, 1]) < 1e-8
    assert rel(Hm[:, 3], Hs[:, 3]) < 1e-8
    bn = np.linalg.norm(b)
    Ax = op.apply(mer.x)
    assert abs(np.linalg.norm(b - Ax) / bn - mer.residual) < 1e-9
    assert np.array_equal(Ax[h.constrained_dofs], mer.x[h.constrained_dofs])
    Ab = op.apply(b)
    assert rel(op.apply(2.0 * mer.x - 3.0 * b), 2.0 * Ax - 3.0 * Ab) < 1e-12
    assert abs(mer.x @ Ax - mer.x @ b) <= 2 * mer.residual * bn * np.linalg.norm(mer.x)
    # symmetry: u.A w == w.A u
    w = np.random.default_rng(9).standard_normal(h.n_dofs)
    w[h.constrained_dofs] = 0.0
    Aw = op.apply(w)
    assert abs(b @ Aw - w @ Ab) <= 1e-11 * np.linalg.norm(b) * np.linalg.norm(Aw)
    # all variants describe the same operator: the first residuals are pinned across variants
    key = [float(v) for v in Hs[:5, 3]]
    seen = _CURVED_SEEN.setdefault("hist", key)
    assert rel(np.array(key), np.array(seen)) < 1e-10


_CURVED_SEEN = {}


@pytest.mark.parametrize("key", ["bp3", "bp4", "bp3_p2"])
def test_bp_canonical_vs_reference(golden, key):
    """BP3 / BP4 exactly as the reference's harness builds them (bench.py:153-187 defaults: mesh deformed by
    0.05, final_tensor_load, n_q = p + 2 Gauss points) against fixtures generated by the unmodified reference
    (oracle/make_golden.py::bp_canonical): manufactured RHS, one apply, the Jacobi diagonal at 1e-12, 25
    iterations of pcg / combined_pcg."""
    from paper_2205_08909_b200 import harness
    S = _solvers()
    g = golden["bp_canonical"]
    bp, p, cells = {"bp3": ("BP3", 5, (3, 3, 3)), "bp4": ("BP4", 5, (2, 2, 3)), "bp3_p2": ("BP3", 2, (4, 3, 5))}[key]
    op, b, minv = harness.assemble_problem(bp, p, cells)
    assert op.spec.n_q_1d == p + 2
    assert rel(b, g[f"{key}_b"]) < 1e-13
    assert rel(op.apply(g[f"{key}_u"]), g[f"{key}_Au"]) < 1e-12
    assert rel(minv.inverse_diagonal, g[f"{key}_invdiag"]) < 1e-12
    for variant in ("pcg", "combined_pcg"):
        res = S.solve(variant, op, g[f"{key}_b"], minv=minv, config=S.SolverConfig(fixed_iterations=25))
        assert rel(hist_array(res.history), g[f"{key}_{variant}_hist"]) < 1e-10, variant
        assert rel(res.x, g[f"{key}_{variant}_x"]) < 1e-10, variant
