"""Pole sharding on one GPU: unreduced pole-shard contexts
(zolo_set_pole_shard without a communicator) return each rank's partial G;
their sum must equal the unsharded G (filter_engine.hpp:63-69, 73-78), the
inner-solve counters must add up, and a 1-rank shard is the plain operator.
A 1-rank NCCL communicator runs the in-library all-reduce path on one GPU.
Multi-rank pole groups run here as threads of one process on one GPU with the
library's collectives staged through the host (zolo_set_pole_shard_host,
sharding.ThreadGroup): the same control flow as NCCL -- pole partition,
row-blocked combine, reduce-scatter, row-sharded CGS2 with all-reduced inner
products, all-gather of the next basis vector -- and no kernel of one rank ever
waits on another's (NCCL itself rejects two ranks on one device).
"""
import os
import subprocess
import sys
import threading

import numpy as np
import pytest

from conftest import golden_pencil, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def zb():
    import paper_1701_08935_b200 as zb

    return zb


@pytest.mark.parametrize("case,nranks", [("filter_cfg2_k6", 2), ("filter_cfg2_k6", 3), ("filter_planted30_cx", 2),
                                         ("filter_cfg3_k5", 4)])
def test_partial_g_sums_to_full(zb, case, nranks):
    g = load_golden(case)
    cx, r = bool(g["cx"]), int(g["r"])
    if r < nranks:
        pytest.skip("needs r >= nranks")
    pen = golden_pencil(g)
    full = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64)
    ref = full.apply_g(g["v"])
    parts, inner = [], 0
    for rank in range(nranks):
        op = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64, shard=(rank, nranks, None))
        assert op.poles == list(range(rank, r, nranks))
        parts.append(op.apply_g(g["v"]))
        inner += op.inner_solve_count()
        with pytest.raises(zb.DomainError):
            op.apply_filter(g["v"])  # an unreduced shard cannot drive GMRES
    tot = parts[0]
    for p in parts[1:]:
        tot = tot + p
    assert np.abs(tot - ref).max() <= 1e-11 * max(1.0, np.abs(ref).max())
    assert inner == full.inner_solve_count()  # (2 if cx else 1) * r per G application


def test_single_rank_shard_is_plain_operator(zb):
    g = load_golden("filter_cfg2_k6")
    cx, r = bool(g["cx"]), int(g["r"])
    pen = golden_pencil(g)
    a = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64)
    b = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64, shard=(0, 1, None))
    ya, _ = a.apply_filter(g["v"])
    yb, _ = b.apply_filter(g["v"])
    assert (ya == yb).all()


def test_one_rank_nccl_communicator(zb):
    """The in-library NCCL path on one GPU: a 1-rank communicator (ncclCommInitRank with nranks=1)
    all-reduces every G application in place; the sum over one rank is the identity, so the filtered
    block, report and counters must equal the plain operator's bit for bit."""
    g = load_golden("filter_planted30_cx")
    cx, r = bool(g["cx"]), int(g["r"])
    pen = golden_pencil(g)
    a = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64)
    b = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64, shard=(0, 1, zb.nccl_unique_id()))
    ya, ra = a.apply_filter(g["v"])
    yb, rb = b.apply_filter(g["v"])
    assert (ya == yb).all()
    assert ra.iterations == rb.iterations and ra.column_iterations == rb.column_iterations
    assert a.inner_solve_count() == b.inner_solve_count() and a.g_application_count() == b.g_application_count()
    assert (a.apply_g(g["v"]) == b.apply_g(g["v"])).all()


def _run_group(zb, case, nranks, refine=0):
    """Filter the golden case's block with a pole group of `nranks` threads (host collectives);
    returns [(y, report, inner, gapps)] per rank."""
    from paper_1701_08935_b200.sharding import ThreadGroup

    g = load_golden(case)
    cx, r = bool(g["cx"]), int(g["r"])
    pen = golden_pencil(g)
    group = ThreadGroup(nranks)
    out = [None] * nranks
    errs = []

    def rank_main(rank):
        try:
            op = zb.FilterOperator(pen, g["design"], r, is_complex=cx, nd_leaf=64,
                                   shard=(rank, nranks, group.callback(rank)), refine=refine)
            y, rep = op.apply_filter(g["v"])
            out[rank] = (y, rep, op.inner_solve_count(), op.g_application_count())
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            group.barrier.abort()

    ts = [threading.Thread(target=rank_main, args=(q,)) for q in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    return g, out


@pytest.mark.parametrize("case,nranks", [("filter_cfg2_k6", 2), ("filter_cfg2_k6", 3), ("filter_cfg3_k5", 2),
                                         ("filter_planted30_cx", 3), ("filter_zero_column", 2)])
def test_pole_group_threads_match_unsharded_filter(zb, case, nranks):
    """A pole group of 2-3 ranks (row-sharded Arnoldi, the default) filters the block like the
    unsharded operator: every rank returns the same bits, Y matches the unsharded Y and the
    reference golden, Krylov dimensions within +-1, counters partitioned over the ranks."""
    g, out = _run_group(zb, case, nranks)
    cx, r = bool(g["cx"]), int(g["r"])
    y0 = out[0][0]
    for y, rep, _, _ in out[1:]:
        assert (y == y0).all()  # identical bits on every rank
        assert rep.column_iterations == out[0][1].column_iterations
    ref = zb.FilterOperator(golden_pencil(g), g["design"], r, is_complex=cx, nd_leaf=64)
    y1, rep1 = ref.apply_filter(g["v"])
    scale = np.linalg.norm(y1)
    if scale > 0:
        assert np.linalg.norm(y0 - y1) <= 1e-11 * scale
        assert np.linalg.norm(y0 - g["y"]) <= 1e-9 * np.linalg.norm(g["y"])
    assert np.abs(np.array(out[0][1].column_iterations) - np.array(rep1.column_iterations)).max() <= 1
    # every rank counts its own poles' solves; together they are the unsharded count
    gapps = out[0][3]
    assert all(o[3] == gapps for o in out)
    assert sum(o[2] for o in out) == (2 if cx else 1) * r * gapps


def test_pole_group_refined_solves(zb):
    """Refinement inside a pole group: each rank refines its own poles' solves."""
    g, out = _run_group(zb, "filter_cfg3_k5", 2, refine=1)
    assert (out[0][0] == out[1][0]).all()
    assert np.linalg.norm(out[0][0] - g["y"]) <= 1e-9 * np.linalg.norm(g["y"])


def test_replicated_and_row_sharded_arnoldi_agree(zb):
    """ZOLO_ROW_SHARD=0 (G all-reduced, every rank orthogonalising all rows) against the default
    row-sharded Arnoldi: same filtered block to rounding (read once per process -> subprocess)."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_sharding import _run_group
import paper_1701_08935_b200 as zb
g, out = _run_group(zb, "filter_cfg2_k6", 2)
np.save(sys.argv[1], out[0][0])
'''
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ys = []
    for rows in ("0", "1"):
        f = tempfile.mktemp(suffix=".npy")
        subprocess.run([sys.executable, "-c", code, f], check=True, cwd=root, timeout=600,
                       env=dict(os.environ, ZOLO_ROW_SHARD=rows))
        ys.append(np.load(f))
    assert np.linalg.norm(ys[0] - ys[1]) <= 1e-11 * np.linalg.norm(ys[1])
