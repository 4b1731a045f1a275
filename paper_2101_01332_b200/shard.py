"""Multi-GPU e-matching shards.

One process per GPU; every rank holds a replica of the e-graph.  Rank ``r``
of ``world`` e-matches only root candidates whose e-class id lies in the
contiguous id range :func:`class_range` of the allocated-node count (class id
= min node id, reference ``egraph.py:64``).  Matches are ordered by
``(eclass, bindings)`` (``egraph.py:107-112``), so the rank-order
concatenation of the ranks' sorted lists *is* the global sorted list
(:func:`concat_rank_matches`): the device exchange is one NCCL all-gather of
packed per-pattern lists plus an in-order unpack (``csrc/shard.cu``).
Apply / rebuild / cycle filtering / greedy then run on identical inputs on
every rank.

``torch.distributed`` is plumbing only: it carries the NCCL unique id from
rank 0 to the others (:func:`attach_group`) and runs the CPU (gloo) tests of
the partition logic.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Sequence, Tuple

from . import _lib


def class_range(n_alloc: int, rank: int, world: int) -> Tuple[int, int]:
    """[lo, hi) of e-class ids owned by ``rank`` (same formula as tsat_shard_range)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return n_alloc * rank // world, n_alloc * (rank + 1) // world


def shard_matches(matches: Sequence, n_alloc: int, rank: int, world: int) -> list:
    """The part of a sorted match list (``Match``-like, ``.eclass`` or tuple
    head) this rank produces."""
    lo, hi = class_range(n_alloc, rank, world)
    return [m for m in matches if lo <= _eclass(m) < hi]


def concat_rank_matches(parts: Sequence[Sequence]) -> list:
    """Global match list from the ranks' lists (rank order)."""
    out: list = []
    for p in parts:
        out.extend(p)
    return out


def _eclass(m) -> int:
    return m.eclass if hasattr(m, "eclass") else m[0]


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 calls this)."""
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    n = C.c_int32()
    st = lib.tsat_nccl_unique_id(buf, 128, C.byref(n))
    if st != 0:
        raise _lib.E.DeviceError(f"tsat_nccl_unique_id failed with status {st}")
    return buf.raw[: n.value]


def attach(eg, rank: int, world: int, uid: bytes = b"") -> None:
    """Make ``eg`` rank ``rank`` of a ``world``-GPU e-matching shard group.
    Without ``uid`` the engine computes its own shard only (no exchange)."""
    lib = _lib.load()
    _lib.check(eg._h, lib.tsat_shard_setup(eg._h, rank, world, uid or None, len(uid)))


_GROUP_UID: dict = {}


def group_uid(group=None) -> bytes:
    """The NCCL unique id of a torch.distributed group (created by its first
    rank once, then cached: every e-graph of the group shares one communicator)."""
    import torch.distributed as dist

    key = id(group)
    if key not in _GROUP_UID:
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        obj: List = [nccl_unique_id() if rank == 0 and world > 1 else b""]
        if world > 1:
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
        _GROUP_UID[key] = obj[0]
    return _GROUP_UID[key]


def attach_group(eg, group=None) -> None:
    """Shard ``eg`` over the ranks of a torch.distributed process group."""
    import torch.distributed as dist

    attach(eg, dist.get_rank(group), dist.get_world_size(group), group_uid(group))


def attach_host(eg, group=None) -> None:
    """Shard ``eg`` over a torch.distributed group whose backend moves HOST
    tensors (gloo): the engine's exchanges (per-pattern match counts, packed
    match lists, greedy wide-level {cost, node} records) go device -> host ->
    ``all_gather`` -> host -> device instead of NCCL.  Several ranks can then
    share one GPU, which is how the exchange is tested on a one-GPU box."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)

    def _allgather(_ctx, send, recv, nbytes):
        try:
            n = int(nbytes)
            src = torch.empty(n, dtype=torch.uint8)
            if n:
                C.memmove(src.data_ptr(), send, n)
            parts = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, src, group=group)
            for r, t in enumerate(parts):
                if n:
                    C.memmove(recv + r * n, t.data_ptr(), n)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the engine as a failed transport
            return 1

    cb = _lib.ALLGATHER_FN(_allgather)
    eg._shard_cb = cb  # keep the trampoline alive as long as the engine
    lib = _lib.load()
    _lib.check(eg._h, lib.tsat_shard_setup_host(eg._h, rank, world, cb, None))


def lib_class_range(n_alloc: int, rank: int, world: int) -> Tuple[int, int]:
    """tsat_shard_range through the C-ABI (pure host function, no device)."""
    lib = _lib.load()
    lo, hi = C.c_uint32(), C.c_uint32()
    st = lib.tsat_shard_range(n_alloc, rank, world, C.byref(lo), C.byref(hi))
    if st != 0:
        raise ValueError("bad rank / world size")
    return lo.value, hi.value
