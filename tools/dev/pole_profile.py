"""development: per-pole min pivot ratio and the poles of a config's filter design."""
import sys

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
pen, cx, gaps, r, nv, nl = configs.config(name)
d = build_filter_design(gaps, r)
op = zb.FilterOperator(pen, d, r, is_complex=cx, block_size=configs.BLOCK_SIZE.get(name, 1))
prof = op.factor_profile()
for j, p in enumerate(prof):
    print(f"{name} pole {j}: sigma = {op.poles[j]:.6e}  min_pivot_ratio {p['min_pivot_ratio']:.3e}")
