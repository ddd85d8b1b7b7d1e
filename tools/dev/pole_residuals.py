"""development: relative residual of the unrefined / refined shifted solves per pole, and the pole weights."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs, design as dz  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
pen, cx, gaps, r, nv, nl = configs.config(name)
n, a, b = pen
d = dz.build_filter_design(gaps, r)
A = sp.csr_matrix((np.asarray(a[2]).view(np.complex128) if cx else a[2], a[1], a[0]), shape=(n, n))
B = sp.identity(n, format="csr") if b is None else sp.csr_matrix(
    (np.asarray(b[2]).view(np.complex128) if cx else b[2], b[1], b[0]), shape=(n, n))
sig = dz.inner_poles(d, r)
w = d[dz.HEAD + 2 * r:dz.HEAD + 4 * r:2] + 1j * d[dz.HEAD + 2 * r + 1:dz.HEAD + 4 * r:2]
op = zb.FilterOperator(pen, d, r, is_complex=cx, block_size=configs.BLOCK_SIZE.get(name, 1))
rng = np.random.default_rng(0)
rhs = rng.standard_normal((n, 4)) + 1j * rng.standard_normal((n, 4))
for refine in (0, 1):
    op.set_refinement(refine)
    for j in range(r):
        x = op.shifted_solve(rhs, pole=j)
        K = A - sig[j] * B
        res = np.linalg.norm(rhs - K @ x) / np.linalg.norm(rhs)
        xs = np.linalg.norm(x) / np.linalg.norm(rhs)
        print(f"{name} refine={refine} pole {j}: sigma={sig[j]:.3e} |w|={abs(w[j]):.3e} residual {res:.2e} |x|/|b| {xs:.2e} "
              f"pivot ratio {op.factor_profile()[j]['min_pivot_ratio']:.2e}", flush=True)
