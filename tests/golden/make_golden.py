"""Generate the golden fixtures in tests/golden/*.npz from the UNMODIFIED
reference library (oracle/_ref/libzoloref.so, built from
/root/reference/proj/include by oracle/Makefile).

Run here (the container that has /root/reference):
    make -C oracle ref && python tests/golden/make_golden.py

Each case mirrors an assertion of the reference's own Catch2 suite (cited
per case) or a BASELINE.json config at oracle-scale size. Every fixture
stores its inputs (pencil, window, order, block) next to the reference's
outputs, so the parity tests need neither /root/reference nor the
generators at run time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
import pencils as P  # noqa: E402


def pack_pencil(prefix, pencil, out):
    n, a, b = pencil
    out[prefix + "n"] = np.int64(n)
    out[prefix + "a_rp"], out[prefix + "a_ci"], out[prefix + "a_v"] = a
    if b is not None:
        out[prefix + "b_rp"], out[prefix + "b_ci"], out[prefix + "b_v"] = b


def save(name, **kw):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def main():
    ref = oracle.Reference()

    # --- designs (filter_design.hpp:133-169; pins test_mobius.cpp:28-35,
    #     test_filter_design.cpp:28-45, criterion 4) ---
    designs = {}
    windows = {
        "fig4_r9": ([-1.1, -0.9, 0.9, 1.1], 9),
        "fig4_r4": ([-1.1, -0.9, 0.9, 1.1], 4),
        "diag10_r3": ([2.0, 3.0, 6.0, 7.0], 3),
        "diag10_r4": ([2.0, 3.0, 6.0, 7.0], 4),
        "planted_r3": ([10.0, 11.0, 20.0, 21.0], 3),
        "leftopen_r4": ([-np.inf, 1.0, 3.0, 5.0], 4),
        "pf_r4": ([-1.3, -0.8, 1.1, 1.7], 4),
        "narrow_r8": ([-1.0005, -0.9995, 0.9995, 1.0005], 8),
    }
    for key, (gaps, r) in windows.items():
        designs["gaps_" + key] = np.asarray(gaps)
        designs["r_" + key] = np.int64(r)
        designs["design_" + key] = ref.design(gaps, r)
        xs = np.linspace(-3, 3, 61)
        xs = xs[np.abs(xs - ref.design(gaps, r)[8]) > 1e-6]
        g, f = ref.eval_scalar(gaps, r, xs)
        designs["x_" + key] = xs
        designs["g_" + key] = g
        designs["filt_" + key] = f
    save("designs", **designs)

    # --- shifted factor solves (band_factor.hpp:53-182; test_sparse.cpp:168-265) ---
    solves = {}
    cases = [
        ("identity9", (9, P.to_csr(np.eye(9), False), None), False, 0.0j, 2, 11),
        ("lap1d50", P.laplacian_1d(50), False, 0.5j, 3, 21),
        ("herm60", P.random_hermitian(60, 13), True, 0.7 + 0.9j, 2, 31),
        ("stencil3d5", P.stencil_3d(5), False, 1.5 + 2.0j, 2, 5),
        ("tb4", P.tight_binding(4), True, 0.3 + 0.4j, 3, 7),
    ]
    for name, pen, cx, sigma, k, seed in cases:
        pen_s = pen
        if name == "identity9":
            # factorize(identity) directly: sigma 0 on A = I -> the identity itself
            pen_s = pen
        rhs = ref.random_block(pen[0], k, seed, cx=True)
        res = ref.shifted_solve(pen_s, cx, sigma, rhs)
        out = {}
        pack_pencil("", pen, out)
        save(f"solve_{name}", cx=np.int64(cx), sigma=np.complex128(sigma), rhs=rhs, x=res["x"], xa=res["xa"],
             perm=res["perm"], bw=np.int64(res["bw"]), min_ratio=np.float64(res["min_ratio"]),
             status=np.int64(res["status"]), **out)
    # zero pivot: [[0,1],[1,0]] -> FactorizationError(pivot_index 0) (test_sparse.cpp:236-245)
    zp = (2, P.to_csr(np.array([[0.0, 1.0], [1.0, 0.0]]), False), None)
    res = ref.shifted_solve(zp, False, 0.0j, np.ones((2, 1), dtype=np.complex128))
    out = {}
    pack_pencil("", zp, out)
    save("solve_zeropivot", cx=np.int64(0), sigma=np.complex128(0), rhs=np.ones((2, 1), dtype=np.complex128),
         status=np.int64(res["status"]), pivot_index=np.int64(res["pivot_index"]), **out)

    # --- apply_g / apply_filter (filter_engine.hpp:56-155; test_filter_engine.cpp) ---
    def filter_case(name, pen, cx, gaps, r, v, gmres_tol=1e-12, gmres_max=50, extra=None):
        g_out, cnt = ref.apply_g(pen, cx, gaps, r, v)
        f = ref.apply_filter(pen, cx, gaps, r, v, gmres_tol, gmres_max)
        out = {}
        pack_pencil("", pen, out)
        if extra:
            out.update(extra)
        save(f"filter_{name}", cx=np.int64(cx), gaps=np.asarray(gaps, dtype=np.float64), r=np.int64(r),
             design=ref.design(gaps, r), v=v, gv=g_out, g_counters=cnt, y=f["y"], status=np.int64(f["status"]),
             column_iterations=f["column_iterations"], residuals=f["residuals"], converged=f["converged"],
             iterations=np.int64(f["iterations"]), operator_applications=np.int64(f["operator_applications"]),
             inner_solves=np.int64(f["inner_solves"]), g_applications=np.int64(f["g_applications"]),
             gmres_tol=np.float64(gmres_tol), gmres_max=np.int64(gmres_max), **out)

    d10 = P.diag_pencil(np.arange(1, 11, dtype=np.float64))
    filter_case("diag10", d10, False, [2.0, 3.0, 6.0, 7.0], 3, np.eye(10, order="F"))
    d8 = P.diag_pencil([0.4, 1.7, 2.2, 3.1, 4.9, 6.6, 7.3, 9.8])
    filter_case("diag8", d8, False, [1.0, 2.0, 5.0, 6.0], 2, np.ones((8, 1), order="F"))

    lam = np.arange(1, 31, dtype=np.float64)
    for cx, seed in ((False, 77), (True, 77)):
        w = ref.random_block(30, 30, seed, cx=cx)
        w = w + 2.0 * np.eye(30)
        pen, ad, bd = P.planted_pencil(lam, w, cx)
        v = ref.random_block(30, 5, 123, cx=cx)
        gaps = [10.0, 11.0, 20.0, 21.0]
        dense_out, _ = ref.dense_filter_oracle(ad, bd, cx, gaps, 3, v)
        filter_case("planted30_" + ("cx" if cx else "real"), pen, cx, gaps, 3, v, extra={"dense_oracle": dense_out})

    # config-shaped, oracle-scale
    s2 = P.stencil_2d(16)
    pen = (256, P.to_csr(s2, False), None)
    ev = np.sort(np.linalg.eigvalsh(s2.toarray()))
    # lowest 8 distinct-gap window (config 1 protocol: a- = -inf)
    gaps = [-np.inf, ev[0], ev[7], ev[8]]
    assert ev[8] > ev[7]
    v = ref.random_block(256, 12, 1, cx=False, orthonormalize=True)
    filter_case("cfg1_k16", pen, False, gaps, 4, v)

    pen = P.stencil_3d(6)
    ev = P.dense_generalized_eigvals(pen)
    gaps = P.window_around(ev, 100, 12)
    v = ref.random_block(pen[0], 8, 1, cx=False, orthonormalize=True)
    filter_case("cfg2_k6", pen, False, gaps, 4, v)

    pen = P.tight_binding(5)
    ev = P.dense_generalized_eigvals(pen)
    gaps = P.window_around(ev, 55, 10)
    v = ref.random_block(pen[0], 6, 1, cx=True, orthonormalize=True)
    filter_case("cfg3_k5", pen, True, gaps, 4, v)

    # GmresError: a budget too small for the window (gmres.hpp:173-180)
    pen = P.stencil_3d(5)
    ev = P.dense_generalized_eigvals(pen)
    gaps = P.window_around(ev, 40, 10)
    v = ref.random_block(pen[0], 3, 5, cx=False, orthonormalize=True)
    filter_case("gmres_fail", pen, False, gaps, 2, v, gmres_tol=1e-12, gmres_max=4)

    # zero column: beta = 0 handled without iterations (gmres.hpp:116-117)
    v = ref.random_block(pen[0], 3, 6, cx=False)
    v[:, 1] = 0.0
    filter_case("zero_column", pen, False, P.window_around(ev, 40, 10), 3, np.asfortranarray(v))

    # --- rayleigh_ritz + subspace_iteration (eigensolver.hpp:105-217) ---
    for name, pen, cx, lo, cnt, over, r in (
        ("cfg1_k16", (256, P.to_csr(P.stencil_2d(16), False), None), False, 0, 8, 4, 4),
        ("cfg2_k6", P.stencil_3d(6), False, 100, 12, 6, 4),
        ("cfg3_k5", P.tight_binding(5), True, 55, 10, 6, 4),
    ):
        ev = P.dense_generalized_eigvals(pen)
        gaps = P.window_around(ev, lo, cnt)
        if lo == 0:
            gaps[0] = -np.inf
        res = ref.subspace_iteration(pen, cx, gaps, cnt, over, r, tol=1e-10, seed=1, want_vectors=True)
        q0 = ref.random_block(pen[0], cnt + over, 1, cx=cx, orthonormalize=True)
        f = ref.apply_filter(pen, cx, gaps, r, q0)
        ritz, small_q = ref.rayleigh_ritz(pen, cx, f["y"])
        out = {}
        pack_pencil("", pen, out)
        save(f"solve_driver_{name}", cx=np.int64(cx), gaps=np.asarray(gaps), r=np.int64(r), n_lambda=np.int64(cnt),
             oversample=np.int64(over), design=ref.design(gaps, r), exact=np.sort(ev)[lo:lo + cnt],
             lambdas=res["lambdas"], vectors=res["vectors"], residual=np.float64(res["residual"]),
             n_iter=np.int64(res["n_iter"]), n_gmres=np.int64(res["n_gmres"]), n_solv=np.int64(res["n_solv"]),
             converged=np.int64(res["converged"]), q0=q0, y1=f["y"], ritz1=ritz, small_q1=small_q, **out)


if __name__ == "__main__":
    main()
