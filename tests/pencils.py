"""Small deterministic test pencils (numpy), mirroring the fixtures the
reference's own tests build:

* ``diag_pencil``        test_filter_engine.cpp:28-34
* ``planted_pencil``     test_filter_engine.cpp:38-65 (A = W diag(lam) W^H, B = W W^H)
* ``laplacian_1d``       test_sparse.cpp:176-192
* ``random_hermitian``   test_sparse.cpp:44-59 (random Hermitian band + shift)
* stencil / tight-binding pencils shaped like BASELINE.json configs 1-3,
  at sizes the CPU oracle finishes in seconds.

A pencil is ``(n, A, B)`` with ``A``/``B`` = ``(rp, ci, vals)`` int64 CSR
(full pattern, sorted columns, explicit zeros dropped: sparse.hpp:56-83) or
``B = None`` for the identity.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def to_csr(m, cx):
    m = sp.csr_matrix(m)
    m.sum_duplicates()
    m.eliminate_zeros()
    m.sort_indices()
    dt = np.complex128 if cx else np.float64
    return (m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data.astype(dt))


def to_dense(csr, n):
    rp, ci, v = csr
    return sp.csr_matrix((v, ci, rp), shape=(n, n)).toarray()


def to_scipy(csr, n):
    rp, ci, v = csr
    return sp.csr_matrix((v, ci, rp), shape=(n, n))


def diag_pencil(d):
    d = np.asarray(d, dtype=np.float64)
    return (len(d), to_csr(sp.diags(d), False), None)


def planted_pencil(lam, w, cx):
    """A = W diag(lam) W^H, B = W W^H, W given (e.g. random_gaussian + 2 I)."""
    lam = np.asarray(lam, dtype=np.float64)
    a = (w * lam) @ w.conj().T
    b = w @ w.conj().T
    a = 0.5 * (a + a.conj().T)
    b = 0.5 * (b + b.conj().T)
    n = len(lam)
    return (n, to_csr(a, cx), to_csr(b, cx)), a, b


def laplacian_1d(n):
    m = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1])
    return (n, to_csr(m, False), None)


def random_hermitian(n, seed, bw=4, cx=True):
    rng = np.random.default_rng(seed)
    m = np.zeros((n, n), dtype=np.complex128 if cx else np.float64)
    for i in range(n):
        for j in range(max(0, i - bw), i):
            if rng.random() < 0.6:
                z = rng.standard_normal() + (1j * rng.standard_normal() if cx else 0)
                m[i, j] = z
                m[j, i] = np.conj(z)
        m[i, i] = rng.standard_normal() * 2
    return (n, to_csr(m, cx), None)


def stencil_2d(k):
    """5-point (4, -1) Dirichlet Laplacian on k x k (config 1 shape)."""
    t = sp.diags([-np.ones(k - 1), 2 * np.ones(k), -np.ones(k - 1)], [-1, 0, 1])
    e = sp.identity(k)
    return sp.kron(t, e) + sp.kron(e, t)


def stencil_3d(k, seed=2, mass=True):
    """7-point Laplacian + U[0,1] diagonal, B = mass (1/2, 1/12) (config 2 shape)."""
    t = sp.diags([-np.ones(k - 1), 2 * np.ones(k), -np.ones(k - 1)], [-1, 0, 1])
    e = sp.identity(k)
    lap = sp.kron(sp.kron(t, e), e) + sp.kron(sp.kron(e, t), e) + sp.kron(sp.kron(e, e), t)
    rng = np.random.default_rng(seed)
    a = lap + sp.diags(rng.random(k ** 3))
    adj = sp.csr_matrix(lap)
    adj.setdiag(0)
    adj.eliminate_zeros()
    b = 0.5 * sp.identity(k ** 3) + (-1.0 / 12.0) * adj if mass else None
    n = k ** 3
    return (n, to_csr(a, False), to_csr(b, False) if b is not None else None)


def tight_binding(k, seed=3, disorder=1.5, overlap=0.05, with_b=True):
    """Complex Hermitian periodic tight-binding (config 3 shape): bonds
    -exp(i theta), on-site U[-w,w], B = I + 0.05 S (S nearest-neighbour SPD,
    off-diagonals U[0,1), diagonal = row sum + 1)."""
    rng = np.random.default_rng(seed)
    n = k ** 3
    idx = np.arange(n).reshape(k, k, k)
    rows, cols, hv, sv = [], [], [], []
    for ax in range(3):
        nb = np.roll(idx, -1, axis=ax)
        i = idx.ravel()
        j = nb.ravel()
        th = rng.random(n) * 2 * np.pi
        h = -np.exp(1j * th)
        s = rng.random(n)
        rows += [i, j]
        cols += [j, i]
        hv += [h, np.conj(h)]
        sv += [s, s]
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    a = sp.coo_matrix((np.concatenate(hv), (rows, cols)), shape=(n, n)).tocsr()
    a = a + sp.diags(rng.uniform(-disorder, disorder, n).astype(np.complex128))
    b = None
    if with_b:
        s = sp.coo_matrix((np.concatenate(sv), (rows, cols)), shape=(n, n)).tocsr()
        s = s + sp.diags(np.asarray(s.sum(axis=1)).ravel() + 1.0)
        b = sp.identity(n, dtype=np.complex128) + overlap * s
    return (n, to_csr(a, True), to_csr(b, True) if b is not None else None)


def dense_generalized_eigvals(pencil):
    from scipy.linalg import eigh

    n, a, b = pencil
    ad = to_dense(a, n)
    bd = to_dense(b, n) if b is not None else np.eye(n)
    return eigh(ad, bd, eigvals_only=True)


def window_around(eigs, lo_index, count):
    """Gap endpoints isolating eigs[lo_index : lo_index+count] (sorted eigs);
    each gap is the full spacing to the neighbouring eigenvalue."""
    e = np.sort(eigs)
    a_minus = -np.inf if lo_index == 0 else e[lo_index - 1]
    a_plus = e[lo_index]
    b_minus = e[lo_index + count - 1]
    b_plus = np.inf if lo_index + count >= len(e) else e[lo_index + count]
    return [a_minus, a_plus, b_minus, b_plus]
