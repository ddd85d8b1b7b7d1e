"""Bitwise determinism of apply_filter on a config (two calls, same operator; and a fresh operator)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1701_08935_b200 as zb
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.design import build_filter_design
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
pen, cx, gaps, r, nv, nl = configs.config(name)
d = build_filter_design(gaps, r)
v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)
op = zb.FilterOperator(pen, d, r, is_complex=cx)
y1, r1 = op.apply_filter(v)
y2, r2 = op.apply_filter(v)
op2 = zb.FilterOperator(pen, d, r, is_complex=cx)
y3, r3 = op2.apply_filter(v)
print(name, "same op bitwise:", bool((y1 == y2).all()), "max diff", float(np.abs(y1 - y2).max()),
      "| fresh op bitwise:", bool((y1 == y3).all()), float(np.abs(y1 - y3).max()), "| iters", r1.iterations, r2.iterations, r3.iterations)
g1 = op.apply_g(v); g2 = op.apply_g(v)
print("apply_g bitwise:", bool((g1 == g2).all()), float(np.abs(g1 - g2).max()))
