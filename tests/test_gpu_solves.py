"""Direct pins of the shifted solves (ShiftedFactor::solve / adjoint_solve,
band_factor.hpp:53-117) through zolo_shifted_solve, after the reference's own
assertions in test_sparse.cpp:168-265 and against its golden solutions
(tests/golden/solve_*.npz, oracle/_ref):

* solutions equal the reference's to 1e-12 (both orderings: ND and the reference's RCM);
* residual ||(A - sigma B) x - b|| <= 1e-10 ||b|| (1D Laplacian at sigma = 0.5i, 3D stencil,
  tight binding), plain and refined;
* adjoint solve = dense adjoint solve <= 1e-10; for a real shift of a Hermitian pencil the
  adjoint solve equals the solve;
* min_pivot_ratio > 1e-8 for imaginary shifts; one ordering shared by all shifts;
* the zero pivot of [[0,1],[1,0]] is reported at index 0 under the reference's RCM order.
"""
import numpy as np
import pytest

from conftest import golden_pencil, load_golden

pytestmark = pytest.mark.gpu

CASES = ["identity9", "lap1d50", "herm60", "stencil3d5", "tb4"]


def one_pole_design(sigma):
    """A packed r = 1 design whose only inner pole is sigma (weight 1): factorization target."""
    d = np.zeros(27)
    d[10] = 1.0  # m_hat
    d[17] = 1.0  # outer M
    d[19], d[20] = sigma.real, sigma.imag
    d[21] = 1.0  # weight
    d[24] = 1.0  # outer partial fraction
    d[26] = 1.0  # outer c -> shifts +-i
    return d


def dense(pen):
    from pencils import to_dense

    n, a, b = pen
    return to_dense(a, n), (to_dense(b, n) if b is not None else np.eye(n))


@pytest.mark.parametrize("ordering", ["nd", "rcm"])
@pytest.mark.parametrize("name", CASES)
def test_solves_match_reference(name, ordering):
    import paper_1701_08935_b200 as zb

    g = load_golden("solve_" + name)
    pen = golden_pencil(g)
    cx, sigma = bool(g["cx"]), complex(g["sigma"])
    op = zb.FilterOperator(pen, one_pole_design(sigma), 1, is_complex=cx, ordering=ordering, nd_leaf=16)
    x = op.shifted_solve(g["rhs"])
    xa = op.shifted_solve(g["rhs"], adjoint=True)
    sc = max(np.abs(g["x"]).max(), 1.0)
    assert np.abs(x - g["x"]).max() <= 1e-12 * sc
    assert np.abs(xa - g["xa"]).max() <= 1e-12 * max(np.abs(g["xa"]).max(), 1.0)
    # test_sparse.cpp residual pins
    a, b = dense(pen)
    k = a - sigma * b
    assert np.linalg.norm(k @ x - g["rhs"]) <= 1e-10 * np.linalg.norm(g["rhs"])
    assert np.linalg.norm(k.conj().T @ xa - g["rhs"]) <= 1e-10 * np.linalg.norm(g["rhs"])
    # dense adjoint oracle (test_sparse.cpp:196-206)
    xd = np.linalg.solve(k.conj().T, g["rhs"])
    assert np.linalg.norm(xa - xd) <= 1e-10 * np.linalg.norm(xd)
    if sigma.imag != 0:
        assert op.factor_profile()[0]["min_pivot_ratio"] > 1e-8  # test_sparse.cpp:248-253
    if ordering == "rcm":  # the reference's ordering and half-bandwidth
        assert op.factor_profile()[0]["bandwidth"] == int(g["bw"])


def test_refined_solves_reduce_the_residual():
    """Residual-correction refinement: the residual of the refined solve is at least as small."""
    import paper_1701_08935_b200 as zb

    g = load_golden("solve_tb4")
    pen = golden_pencil(g)
    sigma = complex(g["sigma"])
    a, b = dense(pen)
    k = a - sigma * b
    res = []
    for refine in (0, 1):
        op = zb.FilterOperator(pen, one_pole_design(sigma), 1, is_complex=True, refine=refine, nd_leaf=16)
        x = op.shifted_solve(g["rhs"])
        res.append(np.linalg.norm(k @ x - g["rhs"]) / np.linalg.norm(g["rhs"]))
    assert res[1] <= 1e-13 and res[1] <= res[0] * 1.0001 + 1e-16


def test_real_shift_adjoint_equals_solve():
    """test_sparse.cpp: for a real shift A - sigma B is Hermitian, so the adjoint solve is the solve."""
    import paper_1701_08935_b200 as zb

    g = load_golden("solve_herm60")
    pen = golden_pencil(g)
    op = zb.FilterOperator(pen, one_pole_design(complex(-7.5, 0.0)), 1, is_complex=True, nd_leaf=16)
    x = op.shifted_solve(g["rhs"])
    xa = op.shifted_solve(g["rhs"], adjoint=True)
    assert np.abs(x - xa).max() <= 1e-12 * np.abs(x).max()


def test_shared_ordering_across_shifts():
    """build_shifted_factors orders once for all shifts (band_factor.hpp:203-204): every pole's
    solve is exact for its own shift on the same device ordering."""
    import paper_1701_08935_b200 as zb
    from paper_1701_08935_b200.design import build_filter_design, inner_poles

    g = load_golden("filter_cfg3_k5")
    pen = golden_pencil(g)
    r = int(g["r"])
    op = zb.FilterOperator(pen, g["design"], r, is_complex=True, nd_leaf=16)
    a, b = dense(pen)
    rhs = np.random.default_rng(3).standard_normal((pen[0], 2)) + 0j
    for j, s in enumerate(inner_poles(g["design"], r)):
        x = op.shifted_solve(rhs, pole=j)
        assert np.linalg.norm((a - s * b) @ x - rhs) <= 1e-10 * np.linalg.norm(rhs)
    del build_filter_design


def test_zero_pivot_index_in_reference_order():
    """test_sparse.cpp:236-245: [[0,1],[1,0]] at sigma = 0 -> FactorizationError(pivot_index 0)
    under the reference's RCM order."""
    import paper_1701_08935_b200 as zb

    g = load_golden("solve_zeropivot")
    with pytest.raises(zb.FactorizationError) as ei:
        zb.FilterOperator(golden_pencil(g), one_pole_design(0j), 1, is_complex=False, ordering="rcm")
    assert ei.value.pivot_index == int(g["pivot_index"]) == 0
