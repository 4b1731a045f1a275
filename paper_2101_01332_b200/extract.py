"""Extraction (reference: pkg/src/tensorsat/extract.py).

``greedy_extract`` runs the min-cost relaxation and the reached-selection
walk on the GPU (``tsat_greedy``, csrc/extract.cu).  ``reconstruct`` and the
selection helpers are host-side format code.  ILP extraction (build_ilp /
solve_ilp / export_lp) is out of scope for the B200 engine.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import Iterable, Mapping, Optional

import numpy as np

from . import _lib
from .egraph import CostVector, EGraph
from .errors import ExtractionError, ReconstructError
from .tensor_lang import SIGNATURES, TensorGraph, ValueKind


@dataclass
class SolverStats:
    nodes_explored: int = 0
    lp_solves: int = 0
    time_s: float = 0.0
    optimal: bool = True
    objective: float = 0.0


@dataclass
class ExtractionResult:
    selection: dict
    total_cost: float
    graph: Optional[TensorGraph] = None
    stats: Optional[SolverStats] = None
    optimal: bool = True


def selection_cost(costs: Mapping, selection: Mapping) -> float:
    return sum(costs[n] for n in set(selection.values()))


def selection_is_acyclic(eg: EGraph, selection: Mapping) -> bool:
    state: dict = {}

    def visit(c) -> bool:
        c = eg.find(c)
        s = state.get(c)
        if s == 2:
            return True
        if s == 1:
            return False
        state[c] = 1
        ok = all(visit(ch) for ch in eg.nodes[selection[c]].children)
        state[c] = 2
        return ok

    try:
        return all(visit(c) for c in selection)
    finally:
        visit = None  # break the recursive closure's cycle (it references eg)


def greedy_extract(eg: EGraph, costs: Mapping, filt: Iterable[int] = ()) -> ExtractionResult:
    """Greedy fixpoint extraction on the GPU (extract.py:120-159)."""
    if eg.root is None:
        raise ExtractionError("e-graph has no root")
    t0 = time.perf_counter()
    eg.set_filter(filt)
    lib = _lib.load()
    n = eg.allocated_nodes
    arr = None
    on_device = isinstance(costs, CostVector) and costs._eg is eg and costs._n == n
    if not on_device:
        arr = np.zeros(max(n, 1), np.float64)
        for nid in np.nonzero(eg._alive_flags())[0]:
            arr[nid] = costs[int(nid)]
    cap = max(eg.num_classes, 1)
    sc = np.zeros(cap, np.uint32)
    sn = np.zeros(cap, np.uint32)
    k = C.c_uint32()
    best = C.c_double()
    rounds = C.c_int64()
    _lib.check(eg._h, lib.tsat_greedy(eg._h, _lib.ptr(arr, C.c_double), _lib.ptr(sc, C.c_uint32),
                                      _lib.ptr(sn, C.c_uint32), C.byref(k), C.byref(best), C.byref(rounds)))
    selection = dict(zip(sc[: k.value].tolist(), sn[: k.value].tolist()))
    if on_device:
        # the reference sums c_i over the Python set of selected nodes (extract.py:112-114)
        total = float(sum(costs.gather(list(set(selection.values()))).tolist()))
    else:
        total = selection_cost(costs, selection)
    stats = SolverStats(nodes_explored=int(rounds.value), time_s=time.perf_counter() - t0)
    return ExtractionResult(selection, total, stats=stats)


def _selected_nodes(eg: EGraph, ids) -> dict:
    """(op atom, canonical children) of the selected e-nodes only: one gather on
    the device instead of materialising the whole e-graph."""
    lib = _lib.load()
    ids = np.array(sorted(set(int(x) for x in ids)), np.uint32)
    n = len(ids)
    op = np.zeros(max(n, 1), np.uint32)
    off = np.zeros(n + 1, np.uint32)
    cap = max(4 * n, 16)
    while True:
        kids = np.zeros(cap, np.uint32)
        nk = C.c_uint64()
        _lib.check(eg._h, lib.tsat_download_nodes(eg._h, n, _lib.ptr(ids, C.c_uint32), _lib.ptr(op, C.c_uint32),
                                                  _lib.ptr(off, C.c_uint32), _lib.ptr(kids, C.c_uint32), cap,
                                                  C.byref(nk)))
        if nk.value <= cap:
            break
        cap = int(nk.value)
    atoms = eg._atom_list
    return {int(x): (atoms[int(op[i])], tuple(int(k) for k in kids[off[i]:off[i + 1]])) for i, x in enumerate(ids)}


def reconstruct(eg: EGraph, selection: Mapping) -> TensorGraph:
    """Materialise a selection as a tensor graph (extract.py:584-639)."""
    if eg.root is None:
        raise ReconstructError("e-graph has no root")
    g = TensorGraph()
    built: dict = {}
    onstack: set = set()
    if any(not 0 <= int(v) < eg.allocated_nodes for v in selection.values()):
        raise ReconstructError("selection names an unknown e-node")
    sel_nodes = _selected_nodes(eg, selection.values())
    keys = np.array([int(c) for c in selection] + [int(eg.root)], np.uint32)
    if (keys >= eg.allocated_nodes).any():
        raise ReconstructError("selection names an unknown e-class")
    found = np.zeros(max(len(keys), 1), np.uint32)
    _lib.check(eg._h, _lib.load().tsat_find_batch(eg._h, len(keys), _lib.ptr(keys, C.c_uint32),
                                                  _lib.ptr(found, C.c_uint32)))
    canon = {int(k): int(f) for k, f in zip(keys[:-1], found[:-1])}
    root_cls = int(found[len(keys) - 1])
    selection = {canon[int(c)]: int(v) for c, v in selection.items()}

    class _EN:
        __slots__ = ("id", "op", "children")

        def __init__(self, nid):
            self.id = nid
            self.op, self.children = sel_nodes[nid]

    def build(cid: int) -> str:
        cid = canon.get(cid, cid)
        if cid in built:
            return built[cid]
        if cid in onstack:
            raise ReconstructError(f"cycle through e-class c{cid}")
        if cid not in selection:
            raise ReconstructError(f"selection misses e-class c{cid}")
        onstack.add(cid)
        en = _EN(selection[cid])
        sig = SIGNATURES.get(en.op) if isinstance(en.op, str) else None
        if sig is None:
            raise ReconstructError(f"e-node n{en.id} ({en.op!r}) is not a graph operator")
        params: dict = {}
        inputs: list = []
        for (arg, kind), ch in zip(sig.args, en.children):
            ch = canon.get(ch, ch)
            if kind in (ValueKind.T, ValueKind.TT):
                inputs.append(build(ch))
            else:
                leaf_id = selection.get(ch)
                if leaf_id is None:
                    raise ReconstructError(f"selection misses parameter class c{ch}")
                leaf = _EN(leaf_id)
                if leaf.children:
                    raise ReconstructError(f"parameter class c{ch} selected a non-literal")
                params[arg] = leaf.op
        onstack.discard(cid)
        name = f"e{cid}"
        g.add(name, en.op, tuple(inputs), **params)
        built[cid] = name
        return name

    root_name = build(root_cls)
    build = None  # break the recursive closure's cycle (it references eg)

    def flat(name: str) -> list:
        nd = g.nodes[name]
        if nd.op != "noop":
            return [name]
        return flat(nd.inputs[0]) + flat(nd.inputs[1])

    g.set_outputs(flat(root_name))
    g.root = root_name
    return g


def build_ilp(*a, **k):
    raise NotImplementedError("ILP extraction is out of scope for the B200 engine (use greedy_extract)")


solve_ilp = export_lp = parse_solution = build_ilp
