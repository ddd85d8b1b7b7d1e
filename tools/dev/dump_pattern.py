"""development: write the union pattern of a BASELINE config for tools/dev/plan_bench."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from paper_1701_08935_b200 import configs  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
pen = configs.config(name)[0]
n, a, b = pen
U = sp.csr_matrix((np.ones(len(a[1])), a[1], a[0]), shape=(n, n))
if b is not None:
    U = U + sp.csr_matrix((np.ones(len(b[1])), b[1], b[0]), shape=(n, n))
U = U.tocsr()
U.sort_indices()
with open(out, "wb") as f:
    np.array([n, U.nnz], dtype=np.int64).tofile(f)
    U.indptr.astype(np.int64).tofile(f)
    U.indices.astype(np.int64).tofile(f)
