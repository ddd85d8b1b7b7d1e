"""Stress of the factorization + refined filter path: repeated fresh factorizations and refined
applications must be bitwise identical (races in the left-looking updates, the split-part
combines, the mask writes or the threaded host setup would show)."""
import sys

sys.path.insert(0, ".")
import paper_1701_08935_b200 as zb  # noqa: E402
from paper_1701_08935_b200 import configs  # noqa: E402
from paper_1701_08935_b200.design import build_filter_design  # noqa: E402

for name, reps in (("cfg2", 8), ("cfg3", 4), ("cfg4s", 3)):
    pen, cx, gaps, r, nv, nl = configs.config(name)
    d = build_filter_design(gaps, r)
    v = zb.random_block(pen[0], min(nv, 64), 7, cx=cx, orthonormalize=True)
    ref = None
    bad = 0
    for k in range(reps):
        op = zb.FilterOperator(pen, d, r, is_complex=cx, block_size=configs.BLOCK_SIZE.get(name, 1))
        op.set_refinement(1)
        try:  # four iterations do not converge: the partial result is what is compared
            y, _ = op.apply_filter(v, gmres_max=4)
        except zb.GmresError as e:
            y = e.y
        if ref is None:
            ref = y
        bad += int(not (y == ref).all())
        del op
    print(f"{name}: {reps} fresh refined factor+filter runs, mismatches {bad}", flush=True)
