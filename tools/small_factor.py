import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
from conftest import load_golden, golden_pencil
import paper_1701_08935_b200 as zb
g=load_golden('filter_cfg2_k6')
op=zb.FilterOperator(golden_pencil(g), g['design'], int(g['r']), is_complex=bool(g['cx']), nd_leaf=64)
print('ok', op.apply_g(g['v']).shape)
