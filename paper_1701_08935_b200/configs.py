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


_UNIFORM = None  # alternative source of the stream (a process that must not load the product library)


def use_uniform_source(fn) -> None:
    """Draw the seeded uniforms from fn(seed, n) instead of the product library's
    zolo_uniform_stream -- bench.py's reference arm passes the reference harness's
    zr_uniform_stream (oracle/_ref), so its process maps no product code. Both are the
    raw mt19937_64 stream (pinned equal in tests/test_host_setup.py)."""
    global _UNIFORM
    _UNIFORM = fn


def uniform(seed: int, n: int) -> np.ndarray:
    if _UNIFORM is not None:
        return np.asarray(_UNIFORM(seed, n), dtype=np.float64)
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


def _gaussian(seed: int, n: int) -> np.ndarray:
    """n standard normal deviates by Box-Muller over the seeded uniform stream."""
    u = uniform(seed, 2 * ((n + 1) // 2))
    u1 = np.maximum(u[0::2], 2.0 ** -53)
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.concatenate([r * np.cos(2 * np.pi * u[1::2]), r * np.sin(2 * np.pi * u[1::2])])
    return z[:n]


def chemistry_pencil(k: int = 20, seed: int = 4, block: int = 13, cutoff: float = 2.5, jitter: float = 0.15,
                     overlap: float = 0.1):
    """Config 4: a chemistry-shaped block-sparse Hermitian pencil (BSR, `block` x `block`
    dense blocks per atom). k^3 atoms on a cubic lattice jittered by U[-jitter, jitter]
    spacings; atoms closer than `cutoff` spacings are coupled. A: off-diagonal blocks
    complex Gaussian x exp(-distance), Hermitian-symmetrised, diagonal blocks Hermitian
    Gaussian. B: the same pattern, off-diagonal blocks overlap x exp(-distance) x complex
    Gaussian (Hermitian), plus a diagonal making every row strictly diagonally dominant
    (so B is Hermitian positive definite). Returns the full-pattern CSR pencil
    (io.bsr_to_csr) of order k^3 * block."""
    from . import io as zio

    na = k ** 3
    g = np.stack(np.meshgrid(np.arange(k), np.arange(k), np.arange(k), indexing="ij"), -1).reshape(-1, 3)
    pos = g + jitter * (2.0 * uniform(seed, 3 * na).reshape(na, 3) - 1.0)
    # neighbour pairs within the cutoff (cell list over the lattice: |di| <= ceil(cutoff) + 1)
    reach = int(np.ceil(cutoff)) + 1
    pairs_i, pairs_j, dist = [], [], []
    for dx in range(-reach, reach + 1):
        for dy in range(-reach, reach + 1):
            for dz in range(0, reach + 1):
                if dz == 0 and (dy < 0 or (dy == 0 and dx <= 0)):
                    continue  # each unordered pair once
                sh = g + np.array([dx, dy, dz])
                ok = np.all((sh >= 0) & (sh < k), axis=1)
                i = np.nonzero(ok)[0]
                j = (sh[ok, 0] * k + sh[ok, 1]) * k + sh[ok, 2]
                d = np.linalg.norm(pos[j] - pos[i], axis=1)
                m = d < cutoff
                pairs_i.append(i[m])
                pairs_j.append(j[m])
                dist.append(d[m])
    pi, pj, pd = (np.concatenate(x) for x in (pairs_i, pairs_j, dist))
    npairs, bs2 = len(pi), block * block
    z = _gaussian(seed + 1, 2 * bs2 * (npairs + na) + 2 * bs2 * npairs)
    za = (z[0:2 * bs2 * npairs:2] + 1j * z[1:2 * bs2 * npairs:2]).reshape(npairs, block, block)
    zd = z[2 * bs2 * npairs:2 * bs2 * (npairs + na)]
    zd = (zd[0::2] + 1j * zd[1::2]).reshape(na, block, block)
    zb = z[2 * bs2 * (npairs + na):]
    zb = (zb[0::2] + 1j * zb[1::2]).reshape(npairs, block, block)
    off_a = za * np.exp(-pd)[:, None, None]
    off_b = overlap * zb * np.exp(-pd)[:, None, None]
    diag_a = 0.5 * (zd + np.conj(np.transpose(zd, (0, 2, 1))))
    # block rows: (i, j) and (j, i) = conjugate transpose, plus the diagonal blocks
    rows = np.concatenate([pi, pj, np.arange(na)])
    cols = np.concatenate([pj, pi, np.arange(na)])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    ba = np.concatenate([off_a, np.conj(np.transpose(off_a, (0, 2, 1))), diag_a])[order]
    bb_off = np.concatenate([off_b, np.conj(np.transpose(off_b, (0, 2, 1))), np.zeros((na, block, block))])
    # strict diagonal dominance of B: diagonal = 1 + sum_j |B_ij| over the row
    rowsum = np.zeros((na, block))
    np.add.at(rowsum, np.concatenate([pi, pj]), np.abs(np.concatenate([off_b, np.conj(np.transpose(off_b, (0, 2, 1)))])).sum(axis=2))
    dd = np.zeros((na, block, block), dtype=np.complex128)
    dd[:, np.arange(block), np.arange(block)] = 1.0 + rowsum
    bb_off[2 * npairs:] = dd
    bb = bb_off[order]
    indptr = np.zeros(na + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    indptr = np.cumsum(indptr)
    a_csr = zio.bsr_to_csr(na, block, indptr, cols, ba, True)
    b_csr = zio.bsr_to_csr(na, block, indptr, cols, bb, True)
    return (na * block, a_csr, b_csr)


def multi_gpu_pencil(k: int = 64, seed: int = 5):
    """Config 5: tight binding as config 3 on a k^3 periodic grid, disorder U[-2, 2], B = I."""
    return tight_binding_pencil(k, seed=seed, disorder=2.0, with_b=False)


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
    # tools/find_window_gpu.py cfg4 0.0 200: chemistry_pencil(20, seed=4), 200 eigenvalues around 0
    "cfg4": {"gaps": [-0.0014473551429546204, -0.0014319087193143789, 0.0014380021788383598, 0.0014440721712162489],
             "count": 200},
    # tools/find_window_gpu.py cfg4s 0.0 32: chemistry_pencil(10, seed=4), 32 eigenvalues around 0
    "cfg4s": {"gaps": [-0.002050713632706902, -0.00195394425863924, 0.0019219309968320887, 0.002050941998095368],
              "count": 32},
    # eigsh k=72 sigma=0 on tight_binding_pencil(20, seed=3, disorder=1.5): the 32 eigenvalues around 0
    "cfg3s": {"gaps": [-0.01663101713848762, -0.016183636199440375, 0.014065304252567426, 0.015125174367574061],
              "count": 32},
    # eigsh k=72 sigma=0 on multi_gpu_pencil(20, seed=5): the 32 eigenvalues around 0
    "cfg5s": {"gaps": [-0.01749621111507395, -0.0170219315255981, 0.018059854034975464, 0.01905197161627576],
              "count": 32},
    # tools/find_window_gpu.py cfg5 0.0 256: multi_gpu_pencil(64, seed=5), 256 eigenvalues around 0
    "cfg5": {"gaps": [-0.004444281498217607, -0.004424367355750291, 0.004403209645170138, 0.004455014820632642],
             "count": 256},
}


# BSR block size of a config's pencil (atoms of 13 rows for the chemistry-shaped configs)
BLOCK_SIZE = {"cfg4": 13, "cfg4s": 13}

# The same generator at a size the reference's CPU path (RCM band LU) finishes in
# seconds: the configs whose reference factorization is infeasible (cfg3: ~0.5-1 h and 99 GB;
# cfg5: ~0.4 TB) are compared with the reference on these siblings instead (the cfg4 generator
# needs ~7 min of reference factorization even at 1000 atoms: no sibling).
SMALL_SIBLING = {"cfg3": "cfg3s", "cfg5": "cfg5s"}


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
    if name == "cfg4":  # ~35 GB of factors per pole: all 8 poles need pole sharding (8 GPUs) or the hybrid solve
        w = WINDOWS["cfg4"]
        return chemistry_pencil(20, seed=4), True, w["gaps"], 8, 256, w["count"]
    if name == "cfg4s":  # config 4's generator at 10^3 atoms (N = 13000): fits one GPU with all 8 poles
        w = WINDOWS["cfg4s"]
        return chemistry_pencil(10, seed=4), True, w["gaps"], 8, 64, w["count"]
    if name == "cfg3s":  # config 3's generator at 20^3 (N = 8000)
        w = WINDOWS["cfg3s"]
        return tight_binding_pencil(20, seed=3, disorder=1.5), True, w["gaps"], 8, 64, w["count"]
    if name == "cfg5s":  # config 5's generator at 20^3 (N = 8000)
        w = WINDOWS["cfg5s"]
        return multi_gpu_pencil(20, seed=5), True, w["gaps"], 8, 64, w["count"]
    if name == "cfg5":
        w = WINDOWS["cfg5"]
        return multi_gpu_pencil(64, seed=5), True, w["gaps"], 8, 320, w["count"]
    raise KeyError(name)
