"""Cycle filtering entry points (reference: pkg/src/tensorsat/cycles.py).

Both run on the GPU (csrc/cycles.cu): ``dfs_get_cycles`` reports the back-edge
cycles of the exact lexicographic DFS from the root; ``break_all_cycles``
filter-lists the newest node of each cycle, pass after pass, until no live
cycle is reachable.
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable, Optional

import numpy as np

from . import _lib

FilterList = set


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
