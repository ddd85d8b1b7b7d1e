"""Residual floor of windows centred at 0 (configs 3 / 5) with and without refined solves."""
import sys
import time

sys.path.insert(0, ".")
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
pen, cx, gaps, r, nv, nl = configs.config(name)
for refine in (["auto", False, True] if len(sys.argv) < 3 else [eval(sys.argv[2])]):
    t0 = time.time()
    res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv - nl, r=r, tol=1e-10, seed=1,
                                                    max_subspace_iters=4, refine=refine), is_complex=cx)
    s = res.stats
    print(f"{name} refine={refine}: converged={res.converged} found={len(res.lambdas)}/{nl} residual={res.residual:.3e} "
          f"rel_lam={res.residual_rel_lambda:.3e} first={s.first_residual:.3e} refined_from={s.refined_from} "
          f"n_iter={s.n_iter} n_gmres={s.n_gmres} t_fact={s.factorization_time:.2f} t_iter={s.iteration_time:.2f} "
          f"wall={time.time() - t0:.1f}", flush=True)
