"""(development) sweep launch time of config cfg on a library variant, results not checked:
python tools/dev/probe_time.py cfg3"""
import sys
import time

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402

name = sys.argv[1]
pen, cx, gaps, r, nv, nl = configs.config(name)
op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx, block_size=configs.BLOCK_SIZE.get(name, 1))
v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)
for rep in range(2):
    try:
        op.apply_filter(v, gmres_max=6)
    except Exception as e:  # noqa: BLE001
        pass
    tm = op.last_timings()
    print(f"{name}: trsm {tm['trsm_ms']:.1f} ms / {tm['trsm_launches']} launches = {tm['trsm_ms'] / max(1, tm['trsm_launches']):.2f} ms per sweep")
