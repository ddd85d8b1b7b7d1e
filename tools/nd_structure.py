"""Block structure of the ND factor of a BASELINE config (zolo_nd_structure, host only).

usage: python tools/nd_structure.py cfg2 [leaf]
"""
import ctypes as C
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 192
pen, cx, gaps, r, nv, nl = configs.config(name)
n, a, b = pen
A = sp.csr_matrix((np.abs(a[2]) + 1, a[1], a[0]), shape=(n, n))
U = (A if b is None else A + sp.csr_matrix((np.abs(b[2]) + 1, b[1], b[0]), shape=(n, n))).tocsr()
U.sort_indices()
out = np.zeros(8, dtype=np.int64)
L = zb.lib()
L.zolo_nd_structure.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
rp, ci = U.indptr.astype(np.int64), U.indices.astype(np.int64)
assert L.zolo_nd_structure(n, rp.ctypes.data, ci.ctypes.data, leaf, out.ctypes.data) == 0
print(f"{name}: n={n} npad={out[0]} block rows={out[1]} offdiag tiles={out[2]} critical path={out[3]} "
      f"trailing dense block={out[4]} node groups={out[5]}")
