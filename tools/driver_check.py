"""End-to-end eigensolver (subspace_iteration on the GPU filter) on a BASELINE
config: time-to-all-eigenpairs (BASELINE metric 2) and the solve statistics.

usage: python tools/driver_check.py cfg2 [tol]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pen, cx, gaps, r, nv, nl = configs.config(name)
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-10
cfg = SolveConfig(n_lambda=nl, oversample_k=nv - nl, r=r, tol=tol, seed=1)
for rep in range(2):
    t0 = time.time()
    res = subspace_iteration(pen, gaps, cfg, is_complex=cx)
    wall = time.time() - t0
    s = res.stats
    print(f"{name}: converged={res.converged} found={len(res.lambdas)}/{nl} residual={res.residual:.2e} "
          f"n_iter={s.n_iter} n_gmres={s.n_gmres} n_solv={s.n_solv} t_fact={s.factorization_time:.3f}s "
          f"t_iter={s.iteration_time:.3f}s time-to-all-eigenpairs={res.time_to_all_eigenpairs:.3f}s (wall {wall:.2f}s)",
          flush=True)
