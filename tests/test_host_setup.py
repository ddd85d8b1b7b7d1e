"""CPU tests of the product's host side (no GPU): the C-ABI library loads and
exports every symbol include/zolo_b200.h declares; the host setup (filter
design, RCM ordering, seeded Gaussian block) reproduces the reference's
golden values."""
import os
import re

import numpy as np
import pytest

from conftest import REPO, golden_pencil, load_golden


def header_symbols():
    src = open(os.path.join(REPO, "include", "zolo_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(zolo_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_1701_08935_b200 as zb

    L = zb.lib()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert b"sm_100a" in L.zolo_version()


def test_library_has_no_unresolved_internal_symbols():
    """Every internal (zolo::) symbol the library references is defined in it: an unresolved one
    only surfaces when the GPU box loads the library (dlopen with immediate binding)."""
    import shutil
    import subprocess

    if not shutil.which("nm"):
        pytest.skip("nm not available")
    lib = os.path.join(REPO, "paper_1701_08935_b200", "libzolo_b200.so")
    out = subprocess.run(["nm", "-D", "--undefined-only", lib], capture_output=True, text=True, check=True).stdout
    bad = [ln for ln in out.splitlines() if "_ZN4zolo" in ln]
    assert not bad, bad


def test_no_device_fails_loudly():
    """Without a GPU the operator must raise, never fall back to the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1701_08935_b200 as zb
    from pencils import diag_pencil

    d = load_golden("designs")
    with pytest.raises(zb.CudaError):
        zb.FilterOperator(diag_pencil(np.arange(1.0, 11.0)), d["design_diag10_r3"], 3)


@pytest.mark.parametrize("key", ["fig4_r9", "fig4_r4", "diag10_r3", "diag10_r4", "planted_r3", "leftopen_r4",
                                 "pf_r4", "narrow_r8"])
def test_design_matches_reference(key):
    from paper_1701_08935_b200.design import build_filter_design, eval_scalar

    d = load_golden("designs")
    r = int(d["r_" + key])
    ours = build_filter_design(d["gaps_" + key], r)
    ref = d["design_" + key]
    # same algorithm, same operation order: agreement to a few ulps
    np.testing.assert_allclose(ours, ref, rtol=1e-13, atol=1e-15)
    g, f = eval_scalar(d["gaps_" + key], r, d["x_" + key])
    np.testing.assert_allclose(g, d["g_" + key], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(f, d["filt_" + key], rtol=1e-12, atol=1e-14)


def test_mobius_pins():
    """test_mobius.cpp:28-35 and criterion 4."""
    from paper_1701_08935_b200.design import ELL1, GAMMA, ALPHA, BETA, build_filter_design

    d = build_filter_design([-1.1, -0.9, 0.9, 1.1], 4)
    assert d[ELL1] == pytest.approx(0.0025125786760090644, abs=1e-12)
    assert d[GAMMA] == pytest.approx(-0.05012562893380048, abs=1e-10)
    assert abs(d[ALPHA]) == pytest.approx(np.sqrt(0.99), abs=1e-10)
    assert abs(d[BETA]) == pytest.approx(np.sqrt(0.99), abs=1e-10)


def test_bad_window_is_domain_error():
    import paper_1701_08935_b200 as zb
    from paper_1701_08935_b200.design import build_filter_design

    with pytest.raises(zb.DomainError):
        build_filter_design([3.0, 2.0, 6.0, 7.0], 3)
    with pytest.raises(zb.DomainError):
        build_filter_design([2.0, 3.0, 6.0, 7.0], 17)


@pytest.mark.parametrize("name", ["lap1d50", "herm60", "stencil3d5", "tb4"])
def test_rcm_matches_reference_ordering(name):
    import paper_1701_08935_b200 as zb
    import scipy.sparse as sp

    g = load_golden("solve_" + name)
    n, a, b = golden_pencil(g)
    # pattern of A - iB (band_factor.hpp:203): union with B, or with I
    am = sp.csr_matrix((np.ones(len(a[1])), a[1], a[0]), shape=(n, n))
    bm = sp.identity(n) if b is None else sp.csr_matrix((np.ones(len(b[1])), b[1], b[0]), shape=(n, n))
    u = (am + bm).tocsr()
    u.sort_indices()
    perm, bw, _ = zb.rcm(n, u.indptr.astype(np.int64), u.indices.astype(np.int64))
    assert (perm == g["perm"]).all()
    assert bw == int(g["bw"])


def test_random_block_is_bit_identical_to_reference():
    import paper_1701_08935_b200 as zb

    g = load_golden("solve_driver_cfg1_k16")
    q0 = zb.random_block(256, 12, 1, cx=False, orthonormalize=True)
    assert (q0 == g["q0"]).all()
    g = load_golden("solve_driver_cfg3_k5")
    q0 = zb.random_block(125, 16, 1, cx=True, orthonormalize=True)
    assert np.abs(q0 - g["q0"]).max() == 0.0


@pytest.mark.parametrize("name,near,chunk,order", [("grid2d", 4, 16, 3), ("grid3d", 4, 16, 3), ("grid3d", 2, 8, 1),
                                                   ("grid3d", 3, 12, 0), ("random", 4, 16, 2)])
def test_dag_schedules_are_complete_and_topological(name, near, chunk, order):
    """The claim-ordered sweep schedules (symbolic.cpp dag_schedule) of the ND factor: one row task
    per block row, every dependency summed exactly once (near in the row task, the rest in chunk
    tasks), every partial slot written once, and every task after the tasks it waits on -- the
    property that lets persistent CTAs claim in order without deadlock (checked in C++ on the host)."""
    import ctypes as C

    import scipy.sparse as sp

    import paper_1701_08935_b200 as zb

    if name == "grid2d":
        k = 40
        t = sp.diags([1.0, 1.0, 1.0], [-1, 0, 1], shape=(k, k))
        m = sp.kron(t, sp.identity(k)) + sp.kron(sp.identity(k), t)
    elif name == "grid3d":
        k = 14
        t = sp.diags([1.0, 1.0, 1.0], [-1, 0, 1], shape=(k, k))
        i = sp.identity(k)
        m = sp.kron(sp.kron(t, i), i) + sp.kron(sp.kron(i, t), i) + sp.kron(sp.kron(i, i), t)
    else:
        rng = np.random.default_rng(7)
        n = 1500
        r = sp.random(n, n, density=0.004, random_state=rng)
        m = r + r.T + sp.identity(n)
    m = sp.csr_matrix(m)
    m.sort_indices()
    rp, ci = m.indptr.astype(np.int64), m.indices.astype(np.int64)
    out = np.zeros(4, dtype=np.int64)
    L = zb.lib()
    L.zolo_dag_schedule_check.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p]
    st = L.zolo_dag_schedule_check(m.shape[0], rp.ctypes.data, ci.ctypes.data, 64, near, chunk, order,
                                   out.ctypes.data)
    assert st == 0
    assert out[0] == 0, f"{out[0]} schedule violations"
    assert out[1] >= 2 * out[3]  # at least one row task per block row and direction
