"""Time repeated apply_g (one G application = all r pole solves) on a config (development)."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
pen, cx, gaps, r, nv, nl = configs.config(name)
op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx)
v = zb.random_block(pen[0], nv, 1, cx=cx)
op.apply_g(v)
t0 = time.time()
sw = []
for _ in range(5):
    op.apply_g(v)
    sw.append(op.last_timings()["trsm_ms"])
print(f"{name} {os.environ.get('ZOLO_LIB_PATH', 'default')}: apply_g {1e3 * (time.time() - t0) / 5:.2f} ms, "
      f"sweeps {min(sw):.3f} ms (min of 5)", flush=True)
