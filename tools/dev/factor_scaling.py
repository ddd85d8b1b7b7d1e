"""development: device time of the numeric factorization of a config for r = 1, 2, 4, 8 poles
(per-pole streams overlap: shows whether the level-scheduled LU is bound by its critical path or by throughput)."""
import sys

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
pen, cx, gaps, r, nv, nl = configs.config(name)
for rr in (1, 2, 4, 8):
    for rep in range(2):
        op = zb.FilterOperator(pen, build_filter_design(gaps, rr), rr, is_complex=cx,
                               block_size=configs.BLOCK_SIZE.get(name, 1))
        ms = op.last_timings()["factor_ms"]
        del op
    print(f"{name} r={rr}: factorization {ms:.1f} ms on the device ({ms / rr:.1f} ms per pole)", flush=True)
