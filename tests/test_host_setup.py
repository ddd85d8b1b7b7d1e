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
    """The Python mirror's own design construction (theta series, analytic extrema) against
    the reference's FilterDesign (tests/golden/designs.npz, made by oracle/_ref)."""
    from paper_1701_08935_b200 import design as D

    d = load_golden("designs")
    r = int(d["r_" + key])
    ours = D.build_filter_design(d["gaps_" + key], r)
    ref = d["design_" + key]
    fin = np.isfinite(ref)
    assert (np.isfinite(ours) == fin).all() and (ours[~fin] == ref[~fin]).all()
    err = np.abs(np.where(fin, ours, 0.0) - np.where(fin, ref, 0.0))
    # per-entry scale: the entry, or for the pole / weight blocks the block's largest magnitude
    scale = np.abs(ref).copy()
    h = D.HEAD
    for lo, hi in ((h, h + 2 * r), (h + 2 * r, h + 4 * r)):
        scale[lo:hi] = np.abs(ref[lo:hi]).max()
    scale = np.where(fin, np.maximum(scale, 1e-300), 1.0)
    # the oscillation widths are differences of nearly equal extremum values (rounding-level for
    # the outer function); delta0 is a sampled maximum: compared separately below
    exact = np.ones(ref.size, dtype=bool)
    exact[[D.INNER_DELTA, D.OUTER_DELTA, D.DELTA0]] = False
    assert (err[exact] <= 1e-12 * scale[exact]).all(), np.argmax(err * exact / scale)
    assert abs(ours[D.INNER_DELTA] - ref[D.INNER_DELTA]) <= 1e-9 * ref[D.INNER_DELTA]
    assert abs(ours[D.OUTER_DELTA] - ref[D.OUTER_DELTA]) <= 1e-13 + 1e-6 * ref[D.OUTER_DELTA]
    assert abs(ours[D.DELTA0] - ref[D.DELTA0]) <= 1e-15 + 0.05 * ref[D.DELTA0]
    g, f = D.eval_scalar(d["gaps_" + key], r, d["x_" + key])
    np.testing.assert_allclose(g, d["g_" + key], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(f, d["filt_" + key], rtol=1e-12, atol=1e-14)


CHOOSE_CASES = [([-1.1, -0.9, 0.9, 1.1], 1e-12), ([2.0, 3.0, 6.0, 7.0], 1e-12), ([-1.0005, -0.9995, 0.9995, 1.0005], 1e-14),
                ([-1.0005, -0.9995, 0.9995, 1.0005], 1e-8), ([-np.inf, 1.0, 3.0, 5.0], 1e-10), ([0.1, 0.2, 0.3, 5.0], 1e-16)]


@pytest.mark.parametrize("gaps, eps", CHOOSE_CASES)
def test_choose_order_gonchar(gaps, eps):
    """choose_order (filter_design.hpp:219-232): smallest r whose Gonchar bound meets eps, equal to
    the reference's choice (oracle/_ref, when built here); the chosen design's measured error is
    then below eps (the bound is an upper bound)."""
    import oracle
    from paper_1701_08935_b200 import design as D

    r = D.choose_order(gaps, eps)
    if oracle.Reference.available():
        assert r == oracle.Reference().choose_order(gaps, eps)[0]
    if r < 8:
        assert D.build_filter_design(gaps, r)[D.DELTA0] <= max(eps, 1e-15)


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


def test_large_random_block_threaded_transform_is_bit_identical_to_reference():
    """Blocks of >= 256 Ki Gaussians take host.cpp's threaded Box-Muller path (raw mt19937_64 stream
    sequential, transform on several threads): same bits as the reference's serial
    random_gaussian (dense.hpp:193-208), digests in tests/golden/rng_block_large.npz."""
    import sys

    import paper_1701_08935_b200 as zb

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden import array_digest

    g = load_golden("rng_block_large")
    assert array_digest(zb.random_block(1 << 20, 5, 7, cx=False)) == g["real"]
    assert array_digest(zb.random_block((1 << 19) + 3, 5, 9, cx=True)) == g["cplx"]
    assert array_digest(zb.random_block(32768, 96, 1, cx=False)) == g["mid"]
    assert array_digest(zb.random_block(40000, 9, 5, cx=True)) == g["mid_cplx"]


@pytest.mark.parametrize("name,near,chunk,order", [("grid2d", 4, 16, 3), ("grid3d", 4, 16, 3), ("grid3d", 2, 8, 1),
                                                   ("grid3d", 3, 12, 0), ("random", 4, 16, 2),
                                                   ("grid3d_wide", 0, 1, 3), ("grid3d_wide", 1, 1, 0)])
def test_dag_schedules_are_complete_and_topological(name, near, chunk, order):
    """The claim-ordered sweep schedules (symbolic.cpp dag_schedule) of the ND factor: one row task
    per block row, every dependency summed exactly once (near in the row task, the rest in chunk
    tasks), every task after the tasks it waits on -- the property that lets persistent CTAs claim
    in order without deadlock -- and the accumulated partial slots: every write a fresh stamp, a
    chunk continuing its own chain, a slot taken over only after the row task that read it last,
    each row task reading the last step of each of its chains (checked in C++ on the host).
    grid3d_wide: one dependency per chunk, so the widest rows need more than 64 chunk steps and
    take extra chains."""
    import ctypes as C

    import scipy.sparse as sp

    import paper_1701_08935_b200 as zb

    if name == "grid2d":
        k = 40
        t = sp.diags([1.0, 1.0, 1.0], [-1, 0, 1], shape=(k, k))
        m = sp.kron(t, sp.identity(k)) + sp.kron(sp.identity(k), t)
    elif name.startswith("grid3d"):
        k = 14 if name == "grid3d" else 22
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


@pytest.mark.parametrize("name", ["grid2d", "grid3d", "torus3d", "random"])
def test_factor_plan_is_complete_and_ordered(name):
    """The left-looking factor plan (symbolic.cpp factor_plan) of the ND factor: every tile is
    completed by exactly one target at its block column's level, with all its contributions
    (L(a,k), U(k,b)), k ascending and on lower levels -- the fixed summation order behind the
    deterministic factors -- also across the parts of split targets, each part read by one combine
    entry; the contributions number sum_k |col(k)|^2 (checked in C++ on the host). torus3d is large
    enough for lists of more than 48 contributions, i.e. split targets."""
    import ctypes as C

    import scipy.sparse as sp

    import paper_1701_08935_b200 as zb

    if name == "grid2d":
        k = 60
        t = sp.diags([1.0, 1.0, 1.0], [-1, 0, 1], shape=(k, k))
        m = sp.kron(t, sp.identity(k)) + sp.kron(sp.identity(k), t)
    elif name == "grid3d":
        k = 14
        t = sp.diags([1.0, 1.0, 1.0], [-1, 0, 1], shape=(k, k))
        i = sp.identity(k)
        m = sp.kron(sp.kron(t, i), i) + sp.kron(sp.kron(i, t), i) + sp.kron(sp.kron(i, i), t)
    elif name == "torus3d":
        k = 26
        t = sp.diags([1.0, 1.0, 1.0], [-1, 0, 1], shape=(k, k)).tolil()
        t[0, k - 1] = t[k - 1, 0] = 1.0
        i = sp.identity(k)
        m = sp.kron(sp.kron(t, i), i) + sp.kron(sp.kron(i, t), i) + sp.kron(sp.kron(i, i), t)
    else:
        rng = np.random.default_rng(11)
        n = 2500
        r = sp.random(n, n, density=0.003, random_state=rng)
        m = r + r.T + sp.identity(n)
    m = sp.csr_matrix(m)
    m.sort_indices()
    rp, ci = m.indptr.astype(np.int64), m.indices.astype(np.int64)
    out = np.zeros(8, dtype=np.int64)
    L = zb.lib()
    L.zolo_factor_plan_check.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    assert L.zolo_factor_plan_check(m.shape[0], rp.ctypes.data, ci.ctypes.data, 64, out.ctypes.data) == 0
    assert out[0] == 0, f"{out[0]} plan violations"
    assert out[1] > 0 and out[2] > 0
    if name == "torus3d":
        assert out[3] > 0 and out[4] > 0, "the torus should split some targets"


def test_uniform_stream_matches_reference_mt19937_64():
    """The product's seeded stream (zolo_uniform_stream, host.cpp) equals the reference's
    std::mt19937_64 raw-bit convention (hamiltonian.hpp:50-53) drawn through oracle/_ref
    (tests/golden/rng_streams.npz), bit for bit."""
    from paper_1701_08935_b200 import configs

    g = load_golden("rng_streams")
    for key in g:
        seed = int(key[4:])
        assert (configs.uniform(seed, g[key].size) == g[key]).all()


@pytest.mark.parametrize("name", ["cfg3gen_k12", "cfg5gen_k16", "cfg4gen_k4"])
def test_config_generators_are_pinned(name):
    """The product's config generators rebuild the exact pencils (and the product's random_block
    the exact start blocks) the reference's golden outputs were computed on."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden import array_digest, pencil_digest

    import paper_1701_08935_b200 as zb
    from paper_1701_08935_b200 import configs

    g = load_golden("gen_" + name)
    if name.startswith("cfg3gen"):
        pen = configs.tight_binding_pencil(12, seed=3, disorder=1.5)
    elif name.startswith("cfg5gen"):
        pen = configs.tight_binding_pencil(16, seed=5, disorder=2.0, with_b=False)
    else:
        pen = configs.chemistry_pencil(4, seed=4)
    assert pencil_digest(pen) == g["pencil_sha256"]
    v = zb.random_block(int(g["n"]), int(g["n_v"]), 1, cx=True, orthonormalize=True)
    assert array_digest(v) == g["v_sha256"]
