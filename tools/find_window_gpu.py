"""Locate a BASELINE window on the GPU by Sylvester-inertia bisection
(paper_1701_08935_b200/slicing.py) and print its gap endpoints for configs.py.

usage: python tools/find_window_gpu.py cfg3|cfg4|cfg4s|cfg5 [center] [count]
"""
import sys
import time

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs, slicing  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
center = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 128
gen = {"cfg3": lambda: configs.tight_binding_pencil(48, seed=3, disorder=1.5),
       "cfg4": lambda: configs.chemistry_pencil(20, seed=4),
       "cfg4s": lambda: configs.chemistry_pencil(10, seed=4),
       "cfg5": lambda: configs.multi_gpu_pencil(64, seed=5)}[name]
t0 = time.time()
pen = gen()
print(f"{name}: generated N={pen[0]} nnz(A)={len(pen[1][2])} in {time.time() - t0:.1f} s", flush=True)
t0 = time.time()
ctr = zb.InertiaCounter(pen, is_complex=True)
k = ctr.count_below(center)
print(f"count_below({center}) = {k} ({time.time() - t0:.1f} s incl. symbolic); structure {ctr.structure()}", flush=True)
t0 = time.time()
k2 = ctr.count_below(center + 1e-3)
print(f"one more count: {time.time() - t0:.2f} s", flush=True)
if len(sys.argv) > 4 and sys.argv[4] == "probe":
    sys.exit(0)
t0 = time.time()
gaps = slicing.window_around(ctr, center, count, width=0.05, rtol=1e-12)
print(f"gaps = {gaps!r}  ({time.time() - t0:.1f} s)", flush=True)
print(f"count_in = {ctr.count_in(0.5 * (gaps[0] + gaps[1]), 0.5 * (gaps[2] + gaps[3]))}")
