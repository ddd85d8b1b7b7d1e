"""BSR pencils (BASELINE config 4's format; north star (3) "CSR/BSR SpMM"): with
``block_size`` the nested dissection runs on the atom graph, atoms stay whole,
and the B products of every G application (filter_engine.hpp:60-80) and the
Rayleigh-Ritz A / B products run on the BSR SpMM kernel. Checked against the
CSR path and the oracle (zolo_oracle.c) on a small config-4-shaped pencil."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import paper_1701_08935_b200 as zb
    from paper_1701_08935_b200 import configs
    from paper_1701_08935_b200.design import build_filter_design

    pen = configs.chemistry_pencil(3, seed=4)  # 27 atoms x 13 = 351 rows, complex Hermitian, SPD B
    gaps = configs.window_by_dense_eigs(pen, lo=150, count=12)
    r = 4
    return zb, pen, gaps, r, build_filter_design(gaps, r)


def test_bsr_apply_g_matches_csr(setup):
    zb, pen, gaps, r, design = setup
    v = zb.random_block(pen[0], 20, 3, cx=True, orthonormalize=True)
    csr = zb.FilterOperator(pen, design, r, is_complex=True, nd_leaf=64)
    bsr = zb.FilterOperator(pen, design, r, is_complex=True, nd_leaf=64, block_size=13)
    assert csr.bsr_info() == (1, 0)
    assert bsr.bsr_info() == (13, 27)  # the device SpMMs run on BSR
    a, b = csr.apply_g(v), bsr.apply_g(v)
    assert np.linalg.norm(a - b) <= 1e-11 * np.linalg.norm(a)


def test_bsr_filter_matches_oracle(setup):
    import oracle

    zb, pen, gaps, r, design = setup
    v = zb.random_block(pen[0], 20, 3, cx=True, orthonormalize=True)
    op = zb.FilterOperator(pen, design, r, is_complex=True, nd_leaf=64, block_size=13)
    y, rep = op.apply_filter(v)
    ref = oracle.Oracle().operator(pen, True, design, r).apply_filter(v)
    assert ref["status"] == 0 and rep.all_converged()
    assert np.linalg.norm(y - ref["y"]) <= 1e-9 * np.linalg.norm(ref["y"])
    assert abs(rep.iterations - ref["iterations"]) <= 1


def test_bsr_projection_matches_dense(setup):
    """The Rayleigh-Ritz projections (zolo_rr_project: Y^H A Y, Y^H B Y) on the BSR SpMM."""
    zb, pen, gaps, r, design = setup
    n, a, b = pen
    import scipy.sparse as sp

    A = sp.csr_matrix((a[2], a[1], a[0]), shape=(n, n)).toarray()
    B = sp.csr_matrix((b[2], b[1], b[0]), shape=(n, n)).toarray()
    y = zb.random_block(n, 16, 5, cx=True)
    op = zb.FilterOperator(pen, design, r, is_complex=True, nd_leaf=64, block_size=13)
    at, bt = op.rr_project(y)
    assert np.abs(at - y.conj().T @ A @ y).max() <= 1e-11 * np.abs(at).max()
    assert np.abs(bt - y.conj().T @ B @ y).max() <= 1e-11 * np.abs(bt).max()
