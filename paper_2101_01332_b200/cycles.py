"""Cycle filtering entry points (reference: pkg/src/tensorsat/cycles.py).

Both run on the GPU (csrc/cycles.cu): ``dfs_get_cycles`` reports the back-edge
cycles of the exact lexicographic DFS from the root; ``break_all_cycles``
filter-lists the newest node of each cycle, pass after pass, until no live
cycle is reachable.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Iterable, Optional, Sequence

import numpy as np

from . import _lib

FilterList = set


def _with_filter(eg, filt):
    eg.set_filter(filt)


def live_adjacency(eg, filt: Iterable[int] = ()) -> dict:
    """Class -> child classes through live, unfiltered e-nodes (reference
    cycles.py:29-39), read from the device class graph (tsat_class_graph)."""
    _with_filter(eg, set(filt))
    lib = _lib.load()
    sizes = np.zeros(2, np.uint32)
    _lib.check(eg._h, lib.tsat_class_graph(eg._h, None, None, None, _lib.ptr(sizes, C.c_uint32)))
    n, ne = int(sizes[0]), int(sizes[1])
    cls = np.zeros(max(n, 1), np.uint32)
    off = np.zeros(n + 1, np.uint32)
    dst = np.zeros(max(ne, 1), np.uint32)
    _lib.check(eg._h, lib.tsat_class_graph(eg._h, _lib.ptr(cls, C.c_uint32), _lib.ptr(off, C.c_uint32),
                                           _lib.ptr(dst, C.c_uint32), _lib.ptr(sizes, C.c_uint32)))
    ids = [int(x) for x in cls[:n]]
    return {ids[i]: {ids[int(j)] for j in dst[off[i]:off[i + 1]]} for i in range(n)}


@dataclass
class DescendantsMap:
    """Transitive closure of the live child relation as bitmasks over class
    positions (reference cycles.py:42-67); ``m`` is its own descendant iff it
    lies on a cycle."""

    index: dict
    masks: list
    order: list

    def reaches(self, frm: int, to: int) -> bool:
        fi, ti = self.index.get(frm), self.index.get(to)
        return fi is not None and ti is not None and bool(self.masks[fi] >> ti & 1)

    def descendants(self, cid: int) -> set:
        fi = self.index.get(cid)
        if fi is None:
            return set()
        m = self.masks[fi]
        return {self.order[i] for i in range(len(self.order)) if m >> i & 1}

    def on_cycle(self, cid: int) -> bool:
        return self.reaches(cid, cid)


def get_descendants(eg, filt: Iterable[int] = ()) -> DescendantsMap:
    """The descendants map of the current e-graph (reference cycles.py:70-148),
    computed on the device as the column-parallel bitset closure
    (csrc/cycles.cu k_close_cols) and returned as the reference's
    DescendantsMap.  O(C^2) bits, like the reference."""
    _with_filter(eg, set(filt))
    lib = _lib.load()
    sizes = np.zeros(2, np.uint32)
    _lib.check(eg._h, lib.tsat_descendants(eg._h, None, None, 0, _lib.ptr(sizes, C.c_uint32)))
    n, words = int(sizes[0]), int(sizes[1])
    cls = np.zeros(max(n, 1), np.uint32)
    bits = np.zeros(max(n * words, 1), np.uint32)
    _lib.check(eg._h, lib.tsat_descendants(eg._h, _lib.ptr(cls, C.c_uint32), _lib.ptr(bits, C.c_uint32), bits.size,
                                           _lib.ptr(sizes, C.c_uint32)))
    order = [int(x) for x in cls[:n]]
    rows = bits[: n * words].reshape(words, n).T.copy() if n else bits[:0].reshape(0, 0)
    masks = [int.from_bytes(rows[i].tobytes(), "little") for i in range(n)]
    return DescendantsMap({c: i for i, c in enumerate(order)}, masks, order)


def will_create_cycle(matched_classes: Sequence[int], target_leaf_classes: Sequence[Iterable[int]],
                      d: DescendantsMap, eg) -> bool:
    """The efficient pre-filter (reference cycles.py:151-169): some leaf of
    target i is, or reaches, the class target i is unioned with."""
    for out, leaves in zip(matched_classes, target_leaf_classes):
        out = eg.find(out)
        for leaf in leaves:
            leaf = eg.find(leaf)
            if leaf == out or d.reaches(leaf, out):
                return True
    return False


def vanilla_check(eg, filt: Iterable[int], apply_fn: Callable) -> bool:
    """Complete per-substitution check (reference cycles.py:248-254): apply on
    a device clone of the e-graph, then the DFS cycle search from the root."""
    scratch = eg.clone()
    apply_fn(scratch)
    return bool(dfs_get_cycles(scratch, filt))


def dfs_get_cycles(eg, filt: Iterable[int] = (), root: Optional[int] = None) -> list:
    old_root = eg.root
    if root is not None:
        eg.root = root
    if eg.root is None:
        raise ValueError("e-graph has no root")
    eg.set_filter(filt)
    lib = _lib.load()
    n = C.c_int64()
    try:
        _lib.check(eg._h, lib.tsat_dfs_cycles(eg._h, None, 0, None, 0, C.byref(n)))
        total = -n.value - 1 if n.value < 0 else 0
        if n.value == 0:
            return []
        ncyc_guess = max(total, 1)
        nodes = np.zeros(max(total, 1), np.uint32)
        off = np.zeros(ncyc_guess + 2, np.uint32)
        _lib.check(eg._h, lib.tsat_dfs_cycles(eg._h, _lib.ptr(nodes, C.c_uint32), len(nodes),
                                              _lib.ptr(off, C.c_uint32), len(off), C.byref(n)))
        return [[int(x) for x in nodes[off[i]:off[i + 1]]] for i in range(n.value)]
    finally:
        if root is not None:
            eg.root = old_root


def resolve_cycle(eg, filt: set, cycle) -> Optional[int]:
    if any(n in filt for n in cycle):
        return None
    newest = max(cycle)
    filt.add(newest)
    return newest


def break_all_cycles(eg, filt: set, root: Optional[int] = None) -> int:
    old_root = eg.root
    if root is not None:
        eg.root = root
    eg.set_filter(filt)
    added = C.c_int64()
    try:
        _lib.check(eg._h, _lib.load().tsat_break_cycles(eg._h, C.byref(added)))
    finally:
        if root is not None:
            eg.root = old_root
    dev = eg.get_filter()
    eg._filt_dev = frozenset(dev)
    filt.update(dev)
    eg._touch()
    return int(added.value)
