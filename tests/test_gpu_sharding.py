"""Pole sharding on one GPU: unreduced pole-shard contexts
(zolo_set_pole_shard without a communicator) return each rank's partial G;
their sum must equal the unsharded G (filter_engine.hpp:63-69, 73-78), the
inner-solve counters must add up, and a 1-rank shard is the plain operator.
A 1-rank NCCL communicator runs the in-library all-reduce path on one GPU;
the multi-rank exchange needs two GPUs (NCCL rejects two ranks on one device)
and its host logic is covered by tests/test_sharding_cpu.py (gloo).
"""
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
