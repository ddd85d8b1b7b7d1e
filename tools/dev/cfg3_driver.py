import sys; sys.path.insert(0,'.')
import numpy as np
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration
pen, cx, gaps, r, nv, nl = configs.config("cfg3")
for tol, its in ((1e-10, 5), (1e-9, 5)):
    res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv-nl, r=r, tol=tol, seed=1, max_subspace_iters=its), is_complex=cx)
    s = res.stats
    print(f"tol {tol}: converged={res.converged} found={len(res.lambdas)} residual={res.residual:.3e} rel_lam={res.residual_rel_lambda:.3e} n_iter={s.n_iter} n_gmres={s.n_gmres} first/last={res.lambdas[0]:.15e} {res.lambdas[-1]:.15e} t={res.time_to_all_eigenpairs:.2f}s", flush=True)
print("gaps", gaps)
