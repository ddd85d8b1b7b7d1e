import os, subprocess, sys, numpy as np
code = r'''
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden, golden_pencil
import paper_1701_08935_b200 as zb
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.design import build_filter_design
out = {}
for case in ["filter_cfg2_k6", "filter_cfg3_k5", "filter_planted30_cx"]:
    g = load_golden(case)
    op = zb.FilterOperator(golden_pencil(g), g["design"], int(g["r"]), is_complex=bool(g["cx"]), nd_leaf=64)
    y, rep = op.apply_filter(g["v"])
    out[case] = y
pen, cx, gaps, r, nv, nl = configs.config("cfg2")
op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx)
v = zb.random_block(pen[0], 8, 1, cx=cx, orthonormalize=True)
out["cfg2"] = op.apply_g(v)
np.savez(sys.argv[1], **out)
'''
res = []
for lib in ["tools/dev/variants/libzolo_oldfac.so", "paper_1701_08935_b200/libzolo_b200.so"]:
    f = f"/tmp/cmp_{len(res)}.npz"
    subprocess.run([sys.executable, "-c", code, f], check=True, env=dict(os.environ, ZOLO_LIB_PATH=lib))
    res.append(np.load(f))
for k in res[0].files:
    print(k, "bitwise equal" if (res[0][k] == res[1][k]).all() else f"DIFFER max {np.abs(res[0][k]-res[1][k]).max():.3e}")
