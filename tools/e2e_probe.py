import sys, time, numpy as np, ctypes as C
sys.path.insert(0, '.')
import torch
import paper_1701_08935_b200 as zb
from paper_1701_08935_b200 import configs
from paper_1701_08935_b200.design import build_filter_design
pen, cx, gaps, r, nv, nl = configs.config('cfg2')
op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx)
n = pen[0]
v = zb.random_block(n, nv, 1, cx=cx, orthonormalize=True)
hv = torch.from_numpy(np.ascontiguousarray(v.T)).pin_memory(); hy = torch.empty_like(hv).pin_memory()
dv = hv.cuda(); dy = torch.empty_like(dv)
def e2e():
    rep = zb._Report(); cols = np.zeros(nv, dtype=np.int64)
    rep.column_iterations = cols.ctypes.data_as(C.POINTER(C.c_int64))
    zb._check(op._h, zb.lib().zolo_apply_filter(op._h, C.c_void_p(hv.data_ptr()), C.c_void_p(hy.data_ptr()), nv, 1e-12, 50, C.byref(rep)))
for k in range(3):
    t=time.time(); op.apply_filter_device(dv.data_ptr(), dy.data_ptr(), nv); torch.cuda.synchronize(); t1=time.time()
    e2e(); t2=time.time()
    print(f"device {1e3*(t1-t):.1f} ms ({op.last_timings()['filter_ms']:.1f}), e2e {1e3*(t2-t1):.1f} ms ({op.last_timings()['filter_ms']:.1f})", flush=True)
