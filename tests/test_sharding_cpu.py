"""Multi-GPU host logic on CPU (world_size 2, gloo): the pole and column
shardings of paper_1701_08935_b200/sharding.py against the oracle.

Pole sharding: G = c v + sum_j (...) over poles
(filter_engine.hpp:63-69, 73-78); each rank's partial sum uses its own poles
(and c v on rank 0 only); the all-reduce of the partials must equal the full
G. Column sharding: columns are independent (filter_engine.hpp:109-111), so a
column-split filter gathered over the ranks equals the full-block filter bit
for bit.
"""
import os
import socket

import numpy as np
import pytest

from conftest import golden_pencil, load_golden

CASES = ["filter_cfg2_k6", "filter_planted30_cx"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_dir):
    import sys

    import torch
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    import oracle
    from paper_1701_08935_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden(case)
        cx, r = bool(g["cx"]), int(g["r"])
        pen = golden_pencil(g)
        v = np.asfortranarray(g["v"])
        o = oracle.Oracle()
        # the setup collective: every rank receives rank 0's id
        uid = sharding.exchange_unique_id(lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        # pole sharding: partial G on this rank's poles, all-reduced
        part = o.operator(pen, cx, sharding.partial_weights(g["design"], r, rank, world), r).apply_g(v)
        flat = np.ascontiguousarray(part.T).ravel()  # column-major order
        t = torch.from_numpy(flat.view(np.float64).copy())
        dist.all_reduce(t)
        gv = t.numpy().view(np.complex128 if cx else np.float64).reshape(v.shape[1], v.shape[0]).T
        # column sharding: this rank's block, gathered
        blk = sharding.column_block(v.shape[1], rank, world)
        y_blk = o.operator(pen, cx, g["design"], r).apply_filter(np.asfortranarray(v[:, blk]))["y"]
        parts = [None] * world
        dist.all_gather_object(parts, (blk.start, y_blk))
        if rank == 0:
            y = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])], axis=1)
            np.savez(os.path.join(out_dir, "out.npz"), gv=gv, y=y)
    finally:
        dist.destroy_process_group()


def test_shard_poles_partition():
    from paper_1701_08935_b200.sharding import shard_poles

    for r in range(1, 17):
        for nranks in range(1, r + 1):
            got = sorted(j for g in range(nranks) for j in shard_poles(r, g, nranks))
            assert got == list(range(r))
            assert all(shard_poles(r, g, nranks) for g in range(nranks))  # r >= nranks: nobody idle


def test_column_block_partition():
    from paper_1701_08935_b200.sharding import column_block

    for nv in (1, 7, 96, 320):
        for nranks in (1, 2, 3, 8):
            cols = [c for g in range(nranks) for c in range(nv)[column_block(nv, g, nranks)]]
            assert cols == list(range(nv))


@pytest.mark.parametrize("case", CASES)
def test_gloo_world2_pole_and_column_sharding(case, tmp_path):
    import torch.multiprocessing as mp

    import oracle

    mp.spawn(_worker, args=(2, _free_port(), case, str(tmp_path)), nprocs=2, join=True)
    out = np.load(tmp_path / "out.npz")
    g = load_golden(case)
    cx, r = bool(g["cx"]), int(g["r"])
    pen = golden_pencil(g)
    v = np.asfortranarray(g["v"])
    op = oracle.Oracle().operator(pen, cx, g["design"], r)
    full = op.apply_g(v)
    gv = out["gv"]
    assert np.abs(gv - full).max() <= 1e-12 * max(1.0, np.abs(full).max())
    y_full = op.apply_filter(v)["y"]
    assert (out["y"] == y_full).all()  # columns are independent: bitwise


def _coll_worker(rank, world, port, out_dir):
    import ctypes as C
    import sys

    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    from paper_1701_08935_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn = sharding.gloo_collective()
        cnt = 5
        res = {}
        # the three operations exactly as the library calls them (include/zolo_b200.h ZOLO_COLL_*)
        a = np.arange(cnt, dtype=np.float64) + 10.0 * rank
        assert fn(0, a.ctypes.data_as(C.POINTER(C.c_double)), cnt, None) == 0
        res["allreduce"] = a.copy()
        b = np.arange(world * cnt, dtype=np.float64) * (rank + 1)
        assert fn(1, b.ctypes.data_as(C.POINTER(C.c_double)), cnt, None) == 0
        res["reduce_scatter"] = b[:cnt].copy()
        c = np.zeros(world * cnt)
        c[rank * cnt:(rank + 1) * cnt] = rank + 0.5
        assert fn(2, c.ctypes.data_as(C.POINTER(C.c_double)), cnt, None) == 0
        res["allgather"] = c.copy()
        np.savez(os.path.join(out_dir, f"coll{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def test_gloo_collective_callback_world2(tmp_path):
    """sharding.gloo_collective: the host-staged collective the library calls through
    zolo_set_pole_shard_host, driven with the library's buffer conventions over gloo."""
    import torch.multiprocessing as mp

    world, cnt = 2, 5
    mp.spawn(_coll_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for rank in range(world):
        d = np.load(tmp_path / f"coll{rank}.npz")
        assert (d["allreduce"] == sum(np.arange(cnt) + 10.0 * q for q in range(world))).all()
        full = sum(np.arange(world * cnt, dtype=np.float64) * (q + 1) for q in range(world))
        assert (d["reduce_scatter"] == full[rank * cnt:(rank + 1) * cnt]).all()
        assert (d["allgather"] == np.repeat(np.arange(world) + 0.5, cnt)).all()


def test_thread_group_collectives():
    """sharding.ThreadGroup (ranks as threads of one process, the GPU tests' pole groups):
    every rank gets the same fixed-order sums."""
    import ctypes as C
    import threading

    from paper_1701_08935_b200.sharding import ThreadGroup

    world, cnt = 3, 4
    grp = ThreadGroup(world)
    out = {}

    def run(rank):
        fn = grp.callback(rank)
        a = np.full(cnt, 0.1 * (rank + 1))
        fn(0, a.ctypes.data_as(C.POINTER(C.c_double)), cnt, None)
        b = np.arange(world * cnt, dtype=np.float64) + rank
        fn(1, b.ctypes.data_as(C.POINTER(C.c_double)), cnt, None)
        c = np.zeros(world * cnt)
        c[rank * cnt:(rank + 1) * cnt] = rank
        fn(2, c.ctypes.data_as(C.POINTER(C.c_double)), cnt, None)
        out[rank] = (a, b[:cnt], c)

    ts = [threading.Thread(target=run, args=(q,)) for q in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for rank in range(world):
        a, b, c = out[rank]
        assert (a == out[0][0]).all()  # bitwise identical on every rank
        assert np.allclose(a, 0.1 + 0.2 + 0.3)
        full = sum(np.arange(world * cnt, dtype=np.float64) + q for q in range(world))
        assert (b == full[rank * cnt:(rank + 1) * cnt]).all()
        assert (c == np.repeat(np.arange(world, dtype=np.float64), cnt)).all()


def test_grid_groups():
    from paper_1701_08935_b200.sharding import grid_groups

    assert grid_groups(8, 2) == [[0, 1], [2, 3], [4, 5], [6, 7]]
    assert grid_groups(8, 8) == [list(range(8))]
    with pytest.raises(ValueError):
        grid_groups(6, 4)
