"""Stress: repeated filters must be bitwise identical (races in the sweep kernels would show)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1701_08935_b200 as zb
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.design import build_filter_design
for name, reps in (("cfg1", 20), ("cfg2", 12), ("cfg3", 3)):
    pen, cx, gaps, r, nv, nl = configs.config(name)
    op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx)
    v = zb.random_block(pen[0], nv, 7, cx=cx, orthonormalize=True)
    y0, _ = op.apply_filter(v)
    bad = 0
    for k in range(reps):
        y, _ = op.apply_filter(v)
        bad += int(not (y == y0).all())
    print(f"{name}: {reps} repeats, mismatches {bad}", flush=True)
