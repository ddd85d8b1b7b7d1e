"""Scalar fill of the ND factor inside its 32x32 tiles (development: how much
of the tile-product work multiplies structural zeros).

usage: python tools/tile_density.py cfg2 [leaf]
"""
import ctypes as C
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 256
pen, cx, gaps, r, nv, nl = configs.config(name)
n, a, b = pen
A = sp.csr_matrix((a[2], a[1], a[0]), shape=(n, n))
B = sp.identity(n, format="csr") if b is None else sp.csr_matrix((b[2], b[1], b[0]), shape=(n, n))
K = (A - (6.0 + 0.05j) * B).tocsr()
U = (abs(A) + abs(B)).tocsr()
U.sort_indices()
pos = np.zeros(n, dtype=np.int64)
npad = np.zeros(1, dtype=np.int64)
L = zb.lib()
L.zolo_nd_order.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
rp = U.indptr.astype(np.int64)
ci = U.indices.astype(np.int64)
assert L.zolo_nd_order(n, rp.ctypes.data, ci.ctypes.data, leaf, pos.ctypes.data, npad.ctypes.data) == 0
order = np.argsort(pos)
Kp = K[order][:, order].tocsc()
lu = spla.splu(Kp, permc_spec="NATURAL", diag_pivot_thresh=0.0, options={"SymmetricMode": True})
assert (lu.perm_r == np.arange(n)).all() and (lu.perm_c == np.arange(n)).all()
Lf = lu.L.tocoo()
p = pos[order]  # padded position of factor row k
rows, cols = p[Lf.row], p[Lf.col]
off = rows // 32 != cols // 32
print(f"{name}: n={n} npad={int(npad[0])} scalar nnz(L) strict={int((Lf.row > Lf.col).sum())}")
ti, tj = rows[off] // 32, cols[off] // 32
key = ti * (npad[0] // 32) + tj
uk, inv = np.unique(key, return_inverse=True)
ntiles = len(uk)
rg = (rows[off] % 32) // 8       # warp row group
kg = (cols[off] % 32) // 4       # DMMA k-step
rmask = np.zeros(ntiles, dtype=np.int64)
kmask = np.zeros(ntiles, dtype=np.int64)
np.bitwise_or.at(rmask, inv, 1 << rg)
np.bitwise_or.at(kmask, inv, 1 << kg)
nnz_t = np.bincount(inv)
pc = lambda m: np.array([bin(x).count("1") for x in m])
print(f"off-diagonal tiles {ntiles}, mean density {nnz_t.mean() / 1024:.3f}")
print(f"k-step fraction (8 per tile) {pc(kmask).mean() / 8:.3f}; row-group fraction (4) {pc(rmask).mean() / 4:.3f}; "
      f"both {np.mean(pc(kmask) * pc(rmask)) / 32:.3f}")
