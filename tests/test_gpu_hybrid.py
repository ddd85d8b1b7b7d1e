"""Hybrid inner solve (BASELINE config 2; zolo_set_solve_mode): one factored
pole, shift-invariant multi-shift GMRES on K_p^{-1} B for the others. The
filter it applies is the same operator, so G and the filtered block must match
the direct solve and the reference goldens within the parity tolerances."""
import numpy as np
import pytest

from conftest import golden_pencil, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zb():
    import paper_1701_08935_b200 as zb

    return zb


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("name", ["cfg2_k6", "cfg1_k16", "cfg3_k5", "planted30_cx", "planted30_real"])
def test_hybrid_matches_goldens(zb, name):
    g = load_golden("filter_" + name)
    cx, r = bool(g["cx"]), int(g["r"])
    pen = golden_pencil(g)
    op = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64, solve="hybrid")
    assert op.poles == [0]
    gv = op.apply_g(g["v"])
    assert rel(gv, g["gv"]) <= 1e-10, rel(gv, g["gv"])
    y, rep = op.apply_filter(g["v"], float(g["gmres_tol"]), int(g["gmres_max"]))
    assert rel(y, g["y"]) <= 1e-9, rel(y, g["y"])
    assert rep.all_converged()
    assert np.abs(np.array(rep.column_iterations) - g["column_iterations"]).max() <= 1


def test_hybrid_other_pole_and_cfg1_full(zb):
    """Factoring a different pole gives the same filter; config 1 at full size."""
    from paper_1701_08935_b200 import configs
    from paper_1701_08935_b200.design import build_filter_design

    pen, cx, gaps, r, nv, nl = configs.config("cfg1")
    design = build_filter_design(gaps, r)
    v = zb.random_block(pen[0], 8, 1, cx=cx, orthonormalize=True)
    y_d, _ = zb.FilterOperator(pen, design, r, is_complex=cx).apply_filter(v)
    for p in (0, 2):
        y_h, _ = zb.FilterOperator(pen, design, r, is_complex=cx, solve="hybrid", hybrid_pole=p).apply_filter(v)
        assert rel(y_h, y_d) <= 1e-9
