"""Hybrid inner solve: inner iteration counts and timing vs the direct solve."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1701_08935_b200 as zb  # noqa: E402
from conftest import golden_pencil, load_golden  # noqa: E402

cases = sys.argv[1:] or ["golden:filter_cfg2_k6", "cfg1", "cfg2"]
for case in cases:
    if case.startswith("golden:"):
        g = load_golden(case[7:])
        pen, cx, r, design, v = golden_pencil(g), bool(g["cx"]), int(g["r"]), g["design"], g["v"]
    else:
        from paper_1701_08935_b200 import configs
        from paper_1701_08935_b200.design import build_filter_design
        pen, cx, gaps, r, nv, nl = configs.config(case)
        design = build_filter_design(gaps, r)
        v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)
    yd, repd = zb.FilterOperator(pen, design, r, is_complex=cx, nd_leaf=64 if case.startswith("golden") else 256).apply_filter(v)
    for p in range(r):
        try:
            op = zb.FilterOperator(pen, design, r, is_complex=cx, nd_leaf=64 if case.startswith("golden") else 256,
                                   solve="hybrid", hybrid_pole=p, inner_max=250)
            t0 = time.time()
            y, rep = op.apply_filter(v)
            t = time.time() - t0
            tm = op.last_timings()
            steps = tm["inner_steps"] / max(tm["operator_applications"], 1)
            print(f"{case} pole {p}: outer iters {rep.iterations}, inner steps per G application per column "
                  f"{steps:.1f}, device {tm['filter_ms']:.1f} ms, rel diff vs direct "
                  f"{np.linalg.norm(y - yd) / np.linalg.norm(yd):.2e}", flush=True)
        except Exception as e:
            print(f"{case} pole {p}: {type(e).__name__}: {e}", flush=True)
