"""development: time-to-all-eigenpairs after a filter operator has run in the same process
(as in bench.py), with the operator kept alive or destroyed first."""
import gc
import sys
import time

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402
from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
keep = len(sys.argv) > 2 and sys.argv[2] == "keep"
pen, cx, gaps, r, nv, nl = configs.config(name)
op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx)
v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)
for _ in range(3):
    op.apply_filter(v)
if not keep:
    del op
    gc.collect()
for rep in range(3):
    t0 = time.time()
    res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv - nl, r=r, tol=1e-10, seed=1),
                             is_complex=cx)
    s = res.stats
    print(f"{name} keep={keep} rep {rep}: t_fact={s.factorization_time:.3f}s t_iter={s.iteration_time:.3f}s "
          f"total={res.time_to_all_eigenpairs:.3f}s filter_device={s.filter_device_ms:.1f} ms wall={time.time() - t0:.2f}s",
          flush=True)
