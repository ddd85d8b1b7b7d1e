"""Multi-GPU plumbing for the filter path.

Two shardings, both one process per GPU:

* **columns** -- the columns of V are independent (one Krylov basis per
  column, filter_engine.hpp:109-111): each rank filters its own column block
  with all r factors and no data-path collective (weak scaling).
* **poles** -- the inner operator is a sum over poles
  (filter_engine.hpp:63-69, 73-78): rank g factors the poles
  j = g, g + nranks, ... and every G application ends with one in-place
  ncclAllReduce(sum) inside the library (zolo_set_pole_shard), so all ranks run
  the same Krylov iteration on the same bits (strong scaling; what configs 4/5
  need when one factor fills a GPU).

torch.distributed only carries the setup: the NCCL unique id is created on
rank 0 and broadcast as a Python object over whatever process group the
caller has (gloo or nccl). With the pole groups of a 2D grid (poles x columns,
:func:`grid_operator`) every column group has its own communicator.

The library's collectives can also be staged through the host
(zolo_set_pole_shard_host): :class:`ThreadGroup` runs several ranks as threads of
one process (one GPU; no kernel of one rank waits on another's, so the ranks'
kernels need not be co-resident), :func:`gloo_collective` over torch.distributed.
Both complete every operation with the same fixed-order sum on every rank.
"""
from __future__ import annotations

import threading
from typing import Sequence

import numpy as np


def shard_poles(r: int, rank: int, nranks: int) -> list:
    """Poles rank `rank` of `nranks` factors: j = rank, rank + nranks, ... < r."""
    if not 0 <= rank < nranks:
        raise ValueError("need 0 <= rank < nranks")
    return list(range(rank, r, nranks))


def column_block(nv: int, rank: int, nranks: int) -> slice:
    """Contiguous column block of rank `rank` when n_v columns are split over the ranks."""
    q, rem = divmod(nv, nranks)
    lo = rank * q + min(rank, rem)
    return slice(lo, lo + q + (1 if rank < rem else 0))


def exchange_unique_id(make_id, group=None) -> bytes:
    """Rank 0 calls make_id(); every rank returns the same bytes (broadcast_object_list)."""
    import torch.distributed as dist

    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def pole_sharded_operator(pencil, design, r: int, is_complex: bool, device: int, group=None, **kw):
    """One pole shard of a multi-GPU FilterOperator over the ranks of `group`
    (collective: every rank of the group calls it)."""
    import torch.distributed as dist

    import paper_1701_08935_b200 as zb

    rank, nranks = dist.get_rank(group), dist.get_world_size(group)
    if nranks > r:
        raise ValueError(f"pole sharding needs r >= ranks (r={r}, ranks={nranks})")
    uid = exchange_unique_id(zb.nccl_unique_id, group) if nranks > 1 else None
    return zb.FilterOperator(pencil, design, r, is_complex=is_complex, device=device, shard=(rank, nranks, uid), **kw)


def partial_weights(design: np.ndarray, r: int, rank: int, nranks: int) -> np.ndarray:
    """The packed design restricted to one pole shard: weights of foreign poles and
    (off rank 0) the constant term zeroed -- G of this design is the rank's
    partial sum (used to check the decomposition against the oracle)."""
    d = np.array(design, dtype=np.float64, copy=True)
    own = set(shard_poles(r, rank, nranks))
    head = 19
    for j in range(r):
        if j not in own:
            d[head + 2 * r + 2 * j] = 0.0
            d[head + 2 * r + 2 * j + 1] = 0.0
    if rank != 0:
        d[13] = 0.0
    return d


def reduce_sum(parts: Sequence[np.ndarray]) -> np.ndarray:
    """Fixed-order sum of the ranks' partials (what the all-reduce computes)."""
    out = np.array(parts[0], copy=True)
    for p in parts[1:]:
        out = out + p
    return out


def _host_collective_step(op, buf, count, nranks, rank, slots, barrier):
    """One host-staged collective for rank `rank` (include/zolo_b200.h ZOLO_COLL_*): slots is
    the group's shared list; sums run in rank order, so every rank gets the same bits."""
    size = count if op == 0 else count * nranks
    arr = np.ctypeslib.as_array(buf, shape=(size,))
    slots[rank] = arr.copy() if op != 2 else arr[rank * count:(rank + 1) * count].copy()
    barrier.wait()
    if op == 0:
        acc = slots[0].copy()
        for p in range(1, nranks):
            acc += slots[p]
        arr[:] = acc
    elif op == 1:
        acc = slots[0][rank * count:(rank + 1) * count].copy()
        for p in range(1, nranks):
            acc += slots[p][rank * count:(rank + 1) * count]
        arr[:count] = acc
    else:
        for p in range(nranks):
            arr[p * count:(p + 1) * count] = slots[p]
    barrier.wait()


class ThreadGroup:
    """A pole group of `nranks` ranks that are threads of this process (zolo_set_pole_shard_host):
    the collectives meet in shared host memory."""

    def __init__(self, nranks: int):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.slots = [None] * nranks

    def callback(self, rank: int):
        import paper_1701_08935_b200 as zb

        def fn(op, buf, count, user):
            try:
                _host_collective_step(op, buf, int(count), self.nranks, rank, self.slots, self.barrier)
                return 0
            except Exception:  # a failed rank must not leave the others waiting
                self.barrier.abort()
                return 1

        return zb.COLLECTIVE_FN(fn)


def gloo_collective(group=None):
    """The library's collectives over torch.distributed (any backend with all_reduce /
    all_gather on CPU tensors, e.g. gloo), for zolo_set_pole_shard_host."""
    import torch
    import torch.distributed as dist

    import paper_1701_08935_b200 as zb

    rank, nranks = dist.get_rank(group), dist.get_world_size(group)

    def fn(op, buf, count, user):
        try:
            count = int(count)
            size = count if op == 0 else count * nranks
            arr = np.ctypeslib.as_array(buf, shape=(size,))
            if op == 0 or op == 1:  # reduce-scatter = all-reduce + own block (gloo has no reduce_scatter)
                t = torch.from_numpy(arr.copy())
                dist.all_reduce(t, group=group)
                if op == 0:
                    arr[:] = t.numpy()
                else:
                    arr[:count] = t.numpy()[rank * count:(rank + 1) * count]
            else:
                parts = [torch.zeros(count, dtype=torch.float64) for _ in range(nranks)]
                dist.all_gather(parts, torch.from_numpy(arr[rank * count:(rank + 1) * count].copy()), group=group)
                for p in range(nranks):
                    arr[p * count:(p + 1) * count] = parts[p].numpy()
            return 0
        except Exception:
            return 1

    return zb.COLLECTIVE_FN(fn)


def grid_groups(world: int, poles_per_group: int):
    """2D grid of `world` ranks: column groups of `poles_per_group` consecutive ranks. Returns
    (the list of rank lists, one per column group)."""
    if world % poles_per_group:
        raise ValueError("the world size must be a multiple of the pole-group size")
    return [list(range(g * poles_per_group, (g + 1) * poles_per_group)) for g in range(world // poles_per_group)]


def grid_operator(pencil, design, r: int, is_complex: bool, device: int, nv: int, poles_per_group: int, **kw):
    """One rank of a 2D poles x columns grid (SURVEY.md §8(e) "2D poles x columns grid"): the
    ranks form world / poles_per_group column groups; a group's ranks shard the poles (their own
    NCCL communicator) and filter the group's column block of the n_v columns (columns are
    independent, filter_engine.hpp:109-111). Collective over the world. Returns
    (operator, column slice of this rank's group)."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    groups = grid_groups(world, poles_per_group)
    mine = None
    for ranks in groups:  # every rank takes part in creating every group
        g = dist.new_group(ranks)
        if rank in ranks:
            mine = g
    cg = rank // poles_per_group
    op = pole_sharded_operator(pencil, design, r, is_complex, device, group=mine, **kw)
    return op, column_block(nv, cg, len(groups))
