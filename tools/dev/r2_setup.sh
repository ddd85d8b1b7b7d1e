ZOLO_SETUP_TIMES=1 python -c "
import sys, time; sys.path.insert(0,'.')
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration
for name in ['cfg3']:
    pen, cx, gaps, r, nv, nl = configs.config(name)
    for k in range(2):
        t0=time.time()
        res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv - nl, r=r, tol=1e-10, seed=1), is_complex=cx)
        print(name, 'wall', round(time.time()-t0,3), 'ttae', round(res.time_to_all_eigenpairs,3), 't_fact', round(res.stats.factorization_time,3), 't_iter', round(res.stats.iteration_time,3), 'iters', res.stats.n_iter, 'n_gmres', res.stats.n_gmres, flush=True)
" 2>&1 | tail -40
