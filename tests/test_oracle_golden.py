"""Pins the C restatement (oracle/zolo_oracle.c) against golden vectors that
the unmodified reference emitted (tests/golden/make_golden.py). Where the
restatement keeps the reference's operation order the match is exact."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_pencil, load_golden

SOLVE_CASES = ["identity9", "lap1d50", "herm60", "stencil3d5", "tb4"]
FILTER_CASES = sorted(os.path.basename(p)[7:-4] for p in glob.glob(os.path.join(GOLDEN, "filter_*.npz")))


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_shifted_solve_matches_reference(oracle_lib, name):
    g = load_golden("solve_" + name)
    res = oracle_lib.shifted_solve(golden_pencil(g), bool(g["cx"]), complex(g["sigma"]), g["rhs"])
    assert res["status"] == 0
    assert (res["perm"] == g["perm"]).all()          # rcm.hpp:69-115 ordering
    assert res["bw"] == int(g["bw"])
    assert res["min_ratio"] == pytest.approx(float(g["min_ratio"]), rel=1e-14)
    np.testing.assert_allclose(res["x"], g["x"], rtol=0, atol=1e-14 * np.abs(g["x"]).max())
    np.testing.assert_allclose(res["xa"], g["xa"], rtol=0, atol=1e-14 * np.abs(g["xa"]).max())


def test_zero_pivot_index(oracle_lib):
    g = load_golden("solve_zeropivot")
    res = oracle_lib.shifted_solve(golden_pencil(g), False, 0j, g["rhs"])
    assert int(g["status"]) == 3 and res["status"] == 3
    assert res["pivot_index"] == int(g["pivot_index"]) == 0  # test_sparse.cpp:236-245


@pytest.mark.parametrize("name", FILTER_CASES)
def test_apply_g_and_filter_match_reference(oracle_lib, name):
    g = load_golden("filter_" + name)
    cx, r = bool(g["cx"]), int(g["r"])
    op = oracle_lib.operator(golden_pencil(g), cx, g["design"], r)
    gv = op.apply_g(g["v"])
    np.testing.assert_allclose(gv, g["gv"], rtol=0, atol=1e-13 * max(1.0, np.abs(g["gv"]).max()))
    assert op.counters() == tuple(int(x) for x in g["g_counters"])
    f = op.apply_filter(g["v"], float(g["gmres_tol"]), int(g["gmres_max"]))
    assert f["status"] == int(g["status"])
    if int(g["status"]) == 4:
        # GmresError: the reference rethrows the first failing column's report
        # (filter_engine.hpp:134-137,153); only the failure itself is comparable.
        assert not f["converged"].all() and not g["converged"].all()
        return
    assert (f["column_iterations"] == g["column_iterations"]).all()
    assert f["iterations"] == int(g["iterations"])
    assert f["operator_applications"] == int(g["operator_applications"])
    assert (f["converged"] == g["converged"]).all()
    np.testing.assert_allclose(f["residuals"], g["residuals"], rtol=1e-10, atol=1e-300)
    if int(g["status"]) == 0:
        scale = max(1.0, np.linalg.norm(g["y"]))
        assert np.linalg.norm(f["y"] - g["y"]) <= 1e-13 * scale
        inner, gapps = op.counters()
        assert gapps - 1 == int(g["g_applications"])  # the apply_g above is one extra call
        assert inner == (2 if cx else 1) * r * gapps


def test_planted_dense_oracle_agrees():
    """criterion 6 / test_filter_engine.cpp:145-159: hybrid == dense ≤ 1e-8 ||V||."""
    for name in ("planted30_real", "planted30_cx"):
        g = load_golden("filter_" + name)
        assert np.linalg.norm(g["y"] - g["dense_oracle"]) <= 1e-8 * np.linalg.norm(g["v"])


def test_design_pins():
    d = load_golden("designs")
    # test_mobius.cpp:28-35
    fig = d["design_fig4_r4"]
    assert fig[9] == pytest.approx(0.0025125786760090644, abs=1e-12)
    assert fig[6] == pytest.approx(-0.05012562893380048, abs=1e-10)
    # test_filter_design.cpp:28-45: r=9 poles on one circle of radius sqrt(0.99)
    r = 9
    d9 = d["design_fig4_r9"]
    poles = d9[19:19 + 2 * r:2] + 1j * d9[20:20 + 2 * r:2]
    center = 0.5 * (d9[7] + d9[8])
    assert (poles.imag > 0).all()
    np.testing.assert_allclose(np.abs(poles - center), 0.5 * abs(d9[7] - d9[8]), rtol=1e-10)
