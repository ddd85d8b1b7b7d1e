import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
pen, cx, gaps, r, nv, nl = configs.config(name)
out = []
for tol in (1e-10, 1e-10, 1e-9):
    res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv-nl, r=r, tol=tol, seed=1, max_subspace_iters=3), is_complex=cx)
    out.append(res.lambdas)
    print(f"tol {tol}: converged={res.converged} found={len(res.lambdas)} residual={res.residual:.3e} n_iter={res.stats.n_iter}", flush=True)
print("run0 == run1:", len(out[0]) == len(out[1]) and bool((out[0] == out[1]).all()))
