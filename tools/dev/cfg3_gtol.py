import sys; sys.path.insert(0,'.')
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration
pen, cx, gaps, r, nv, nl = configs.config("cfg3")
for gt in (1e-13, 1e-14):
    res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv-nl, r=r, tol=1e-10, seed=1, max_subspace_iters=4, gmres_tol=gt), is_complex=cx)
    print(f"gmres_tol {gt}: converged={res.converged} residual={res.residual:.3e} rel_lam={res.residual_rel_lambda:.3e} n_iter={res.stats.n_iter} n_gmres={res.stats.n_gmres} min|lam|={min(abs(res.lambdas)):.3e} t={res.time_to_all_eigenpairs:.2f}", flush=True)
