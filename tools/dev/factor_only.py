"""development: one filter operator construction (setup + numeric factorization) of a config, for profiling."""
import sys

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
r_override = int(sys.argv[2]) if len(sys.argv) > 2 else None
pen, cx, gaps, r, nv, nl = configs.config(name)
r = r_override or r
op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx, block_size=configs.BLOCK_SIZE.get(name, 1))
print(f"{name} r={r}: factorization {op.last_timings()['factor_ms']:.1f} ms on the device")
