"""Locate a BASELINE window on the GPU by Sylvester-inertia bisection
(paper_1701_08935_b200/slicing.py) and print its gap endpoints for configs.py.

usage: python tools/find_window_gpu.py cfg3 [center] [count]
"""
import sys
import time

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs, slicing  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
center = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 128
gen = {"cfg3": lambda: (configs.tight_binding_pencil(48, seed=3, disorder=1.5), True)}[name]
pen, cx = gen()
t0 = time.time()
ctr = zb.InertiaCounter(pen, is_complex=cx)
k = ctr.count_below(center)
print(f"{name}: N={pen[0]} count_below({center}) = {k} ({time.time() - t0:.1f} s incl. symbolic)", flush=True)
t0 = time.time()
gaps = slicing.window_around(ctr, center, count, width=0.05, rtol=1e-12)
print(f"gaps = {gaps!r}  ({time.time() - t0:.1f} s)", flush=True)
print(f"count_in = {ctr.count_in(0.5 * (gaps[0] + gaps[1]), 0.5 * (gaps[2] + gaps[3]))}")
