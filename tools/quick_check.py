"""Quick GPU sanity + timing on configs 1 and 2 (development helper)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg2"]:
    pen, cx, gaps, r, nv, nl = configs.config(name)
    design = build_filter_design(gaps, r)
    t0 = time.time()
    order = os.environ.get("ORDER", "nd")
    op = zb.FilterOperator(pen, design, r, is_complex=cx, ordering=order, nd_leaf=int(os.environ.get("ND_LEAF", "192")),
                           block_size=configs.BLOCK_SIZE.get(name, 1))
    t1 = time.time()
    prof = op.factor_profile()[0]
    print(f"{name} [{order}]: N={pen[0]} bw={prof['bandwidth']} factor wall {t1 - t0:.2f}s device {op.last_timings()['factor_ms']:.1f} ms"
          f" min_pivot_ratio {min(p['min_pivot_ratio'] for p in op.factor_profile()):.3e}", flush=True)
    sp = op.sweep_profile()
    print(f"  sweep profile: {sp}", flush=True)
    v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)
    for rep_i in range(2):
        t0 = time.time()
        y, rep = op.apply_filter(v)
        t1 = time.time()
        tm = op.last_timings()
        print(f"  apply_filter wall {t1 - t0:.3f}s device {tm['filter_ms']:.1f} ms trsm {tm['trsm_ms']:.1f} ms"
              f" ({tm['trsm_launches']} launches) iters {rep.iterations} min_col {min(rep.column_iterations)}"
              f" -> {nv / (tm['filter_ms'] / 1e3):.1f} vec/s; iterations {tm['iterations_ms']:.1f} ms on device"
              f" (aux {tm['iterations_ms'] - tm['trsm_ms']:.1f} ms, outside {tm['filter_ms'] - tm['iterations_ms']:.1f} ms)",
              flush=True)
        flops = tm["operator_applications"] * r * (2 if cx else 1) * 2 * (sp["offdiag_tiles"] + sp["block_rows"]) * 8192.0
        print(f"  solve: {flops / (tm['trsm_ms'] * 1e-3) / 1e12:.1f} TF/s over stored tiles", flush=True)
    if name == "cfg1" or os.environ.get("CHECK_ORACLE"):
        import oracle
        if oracle.Reference.available():
            t0 = time.time()
            ref = oracle.Reference().apply_filter(pen, cx, gaps, r, v, threads=os.cpu_count())
            err = np.linalg.norm(y - ref["y"]) / np.linalg.norm(ref["y"])
            print(f"  vs reference ({os.cpu_count()} thr, {time.time() - t0:.1f}s): rel_fro {err:.3e}, "
                  f"ref iters {ref['iterations']}, ref t_filter {ref['t_filter']:.2f}s", flush=True)
