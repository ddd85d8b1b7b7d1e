"""Synthetic pencils of the BASELINE.json configs (the reference ships no
generators for them; SURVEY.md §8(d) "Config generators" fixes the recipe).

Disorder follows the reference's RNG convention: raw mt19937_64 bits scaled
as (x >> 11) 2^-53 (hamiltonian.hpp:52), through the C ABI so a C++ user of
the reference can regenerate the identical pencil. Pencils are
``(n, A, B)`` with int64 CSR (full pattern, sorted columns) and ``B = None``
for the identity -- the SparsePencil<S> layout (sparse.hpp:133-150).

Windows (gap endpoints) for configs 2-5 cannot be known analytically; they
were located once by shift-invert Lanczos (scipy ``eigsh``) with
``tools/find_windows.py`` and are recorded in ``WINDOWS`` below, so the bench
needs no eigensolver at run time. The eigenvalue count inside each window is
re-checked by the solver's own result (north_star: "count must match").
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import _ptr, lib


def uniform(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    lib().zolo_uniform_stream(seed, n, _ptr(out))
    return out


def to_csr(m, cx=False):
    m = sp.csr_matrix(m)
    m.sum_duplicates()
    m.eliminate_zeros()
    m.sort_indices()
    dt = np.complex128 if cx else np.float64
    return (m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data.astype(dt))


def _lap1d(k):
    return sp.diags([-np.ones(k - 1), 2.0 * np.ones(k), -np.ones(k - 1)], [-1, 0, 1])


def stencil2d_pencil(k: int = 64):
    """Config 1: 5-point Laplacian (4 on the diagonal, -1 per neighbour) on a
    k x k Dirichlet grid, B = I."""
    t, e = _lap1d(k), sp.identity(k)
    a = sp.kron(t, e) + sp.kron(e, t)
    return (k * k, to_csr(a), None)


def stencil2d_eigs(k: int = 64):
    """4 sin^2(i pi/(2(k+1))) + 4 sin^2(j pi/(2(k+1))), ascending."""
    i = np.arange(1, k + 1)
    s = 4 * np.sin(i * np.pi / (2 * (k + 1))) ** 2
    return np.sort((s[:, None] + s[None, :]).ravel())


def stencil3d_pencil(k: int = 32, seed: int = 2):
    """Config 2: 7-point Laplacian (6, -1) + diag U[0,1] (seeded) on k^3 Dirichlet;
    B = 7-point mass matrix (1/2 on the diagonal, 1/12 per neighbour), SPD."""
    t, e = _lap1d(k), sp.identity(k)
    lap = sp.kron(sp.kron(t, e), e) + sp.kron(sp.kron(e, t), e) + sp.kron(sp.kron(e, e), t)
    n = k ** 3
    a = lap + sp.diags(uniform(seed, n))
    adj = sp.csr_matrix(lap)
    adj.setdiag(0)
    adj.eliminate_zeros()
    b = 0.5 * sp.identity(n) + (-1.0 / 12.0) * adj  # adj holds -1 per neighbour
    return (n, to_csr(a), to_csr(b))


def tight_binding_pencil(k: int, seed: int = 3, disorder: float = 1.5, overlap: float = 0.05, with_b: bool = True):
    """Configs 3 / 5: complex Hermitian tight binding on a k^3 periodic grid.
    Bonds -exp(i theta), theta ~ U[0, 2 pi); on-site U[-w, w]; B = I + 0.05 S with
    S a nearest-neighbour SPD overlap (off-diagonals U[0,1), diagonal = row sum + 1),
    or B = I (config 5)."""
    n = k ** 3
    u = uniform(seed, 3 * n * 2 + n)
    idx = np.arange(n).reshape(k, k, k)
    rows, cols, hv, sv = [], [], [], []
    for ax in range(3):
        i = idx.ravel()
        j = np.roll(idx, -1, axis=ax).ravel()
        th = 2.0 * np.pi * u[(2 * ax) * n:(2 * ax + 1) * n]
        s = u[(2 * ax + 1) * n:(2 * ax + 2) * n]
        h = -np.exp(1j * th)
        rows += [i, j]
        cols += [j, i]
        hv += [h, np.conj(h)]
        sv += [s, s]
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    a = sp.coo_matrix((np.concatenate(hv), (rows, cols)), shape=(n, n)).tocsr()
    onsite = disorder * (2.0 * u[6 * n:7 * n] - 1.0)
    a = a + sp.diags(onsite.astype(np.complex128))
    b = None
    if with_b:
        s = sp.coo_matrix((np.concatenate(sv), (rows, cols)), shape=(n, n)).tocsr()
        s = s + sp.diags(np.asarray(s.sum(axis=1)).ravel() + 1.0)
        b = to_csr(sp.identity(n, dtype=np.complex128) + overlap * s, True)
    return (n, to_csr(a, True), b)


def window_by_dense_eigs(pencil, lo: int, count: int):
    """Gap endpoints isolating eigenvalues lo..lo+count-1 (dense; small pencils)."""
    from scipy.linalg import eigh

    n, a, b = pencil
    ad = sp.csr_matrix((a[2], a[1], a[0]), shape=(n, n)).toarray()
    bd = np.eye(n) if b is None else sp.csr_matrix((b[2], b[1], b[0]), shape=(n, n)).toarray()
    e = np.sort(eigh(ad, bd, eigvals_only=True))
    return [-np.inf if lo == 0 else e[lo - 1], e[lo], e[lo + count - 1], np.inf if lo + count >= n else e[lo + count]]


# Gap endpoints (a-, a+, b-, b+) per config; see tools/find_windows.py.
WINDOWS = {
    # eigsh k=140 sigma=6.0 on stencil3d_pencil(32, seed=2): 64 eigenvalues near 6,
    # relative eigengap 2.44e-2 (SURVEY.md §8(d) probe: 2.4e-2, m = 21-22)
    "cfg2": {"gaps": [5.988587801896479, 5.989530607165887, 6.0273252122304335, 6.0282488360560285], "count": 64},
    # tools/find_window_gpu.py cfg3 0.0 128 (Sylvester-inertia bisection on the B200, rtol 1e-12):
    # the 128 eigenvalues of tight_binding_pencil(48, seed=3, disorder=1.5) around 0
    "cfg3": {"gaps": [-0.004303539789179923, -0.004240734865379634, 0.004296055916711339, 0.004322829099328374],
             "count": 128},
}


def config(name: str):
    """(pencil, is_complex, gaps, r, n_v, n_lambda) for a BASELINE config."""
    if name == "cfg1":
        lam = stencil2d_eigs(64)
        return stencil2d_pencil(64), False, [-np.inf, lam[0], lam[31], lam[32]], 4, 48, 32
    if name == "cfg2":
        w = WINDOWS["cfg2"]
        return stencil3d_pencil(32, seed=2), False, w["gaps"], 4, 96, w["count"]
    if name == "cfg3":
        w = WINDOWS["cfg3"]
        return tight_binding_pencil(48, seed=3, disorder=1.5), True, w["gaps"], 8, 192, w["count"]
    raise KeyError(name)
