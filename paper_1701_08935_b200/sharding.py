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
caller has (gloo or nccl).
"""
from __future__ import annotations

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
