"""Eigenvalue counting by Sylvester inertia on the GPU (SURVEY.md §8(f) rank 1,
zolo_count_below): counts below / inside windows must equal the exact counts
from dense eigenvalues (small pencils), the analytic spectrum (config 1, full
size) and the configured window count (config 2, 64 eigenvalues)."""
import numpy as np
import pytest
import scipy.linalg as sla

from conftest import golden_pencil, load_golden
from pencils import to_scipy

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zb():
    import paper_1701_08935_b200 as zb

    return zb


def dense_eigs(pen, cx):
    n = pen[0]
    a = to_scipy(pen[1], n).toarray()
    b = to_scipy(pen[2], n).toarray() if pen[2] is not None else np.eye(n)
    return np.sort(sla.eigh(a, b, eigvals_only=True))


@pytest.mark.parametrize("case", ["filter_cfg2_k6", "filter_cfg1_k16", "filter_cfg3_k5", "filter_planted30_cx",
                                  "solve_herm60"])
def test_counts_match_dense_spectrum(zb, case):
    g = load_golden(case)
    cx = bool(g["cx"]) if "cx" in g else np.iscomplexobj(g["a_v"])
    pen = golden_pencil(g)
    lam = dense_eigs(pen, cx)
    ctr = zb.InertiaCounter(pen, is_complex=cx, nd_leaf=64)
    rng = np.random.default_rng(7)
    gaps = np.where(np.diff(lam) > 1e-6 * max(1.0, np.abs(lam).max()))[0]
    picks = rng.choice(gaps, size=min(12, len(gaps)), replace=False)
    sigmas = [0.5 * (lam[k] + lam[k + 1]) for k in picks] + [lam[0] - 1.0, lam[-1] + 1.0]
    for s in sigmas:
        assert ctr.count_below(s) == int(np.sum(lam < s)), s
    a, b = sorted(rng.choice(sigmas, 2, replace=False))
    assert ctr.count_in(a, b) == int(np.sum((lam > a) & (lam < b)))


def test_cfg1_full_size_analytic_counts(zb):
    from paper_1701_08935_b200 import configs

    pen, cx, gaps, r, nv, nl = configs.config("cfg1")
    lam = configs.stencil2d_eigs(64)
    ctr = zb.InertiaCounter(pen, is_complex=cx)
    u = np.unique(np.round(lam, 12))
    for k in (0, 31, 500, 1024, 1800, len(u) - 2):
        s = 0.5 * (u[k] + u[k + 1])
        assert ctr.count_below(s) == int(np.sum(lam < s))
    # the configured window: the lowest 32 (gaps[1] = lam[0], gaps[2..3] bracket the cut)
    assert ctr.count_in(0.5 * lam[0], 0.5 * (lam[31] + lam[32])) == 32
    # the window as configured: a_- = -inf (window.hpp allows one infinite end)
    assert gaps[0] == -np.inf
    assert ctr.count_in(0.5 * (gaps[0] + gaps[1]), 0.5 * (gaps[2] + gaps[3])) == 32
    assert ctr.count_in(-np.inf, np.inf) == pen[0]


def test_cfg2_window_count(zb):
    from paper_1701_08935_b200 import configs

    pen, cx, gaps, r, nv, nl = configs.config("cfg2")
    ctr = zb.InertiaCounter(pen, is_complex=cx)
    a = 0.5 * (gaps[0] + gaps[1])
    b = 0.5 * (gaps[2] + gaps[3])
    assert ctr.count_in(a, b) == nl == 64


def test_cfg2_window_located_by_bisection(zb):
    """The config-2 window gaps (tools/find_windows.py, scipy shift-invert) found
    again from inertia counts alone."""
    from paper_1701_08935_b200 import configs, slicing

    pen, cx, gaps, r, nv, nl = configs.config("cfg2")
    ctr = zb.InertiaCounter(pen, is_complex=cx)
    center = 0.5 * (gaps[1] + gaps[2])
    k0 = ctr.count_below(0.5 * (gaps[0] + gaps[1]))
    got = slicing.window_at(ctr, k0, nl, center, width=0.05, rtol=1e-11)
    assert ctr.count_in(0.5 * (got[0] + got[1]), 0.5 * (got[2] + got[3])) == nl
    np.testing.assert_allclose(got, gaps, rtol=1e-9)
