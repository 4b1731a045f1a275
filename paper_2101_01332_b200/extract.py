"""Extraction (reference: pkg/src/tensorsat/extract.py).

``greedy_extract`` runs the min-cost relaxation and the reached-selection
walk on the GPU (``tsat_greedy``, csrc/extract.cu).  ``reconstruct`` and the
selection helpers are host-side format code.  The ILP model skeleton is
built on the GPU (``tsat_ilp_build``, csrc/ilp.cu); rows / LP text are
host formatting and the MILP solve is scipy (HiGHS).
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


# --------------------------------------------------------------- ILP model
#
# The model skeleton (reachable classes, x variables, live members, distinct
# child classes per live member) is built on the GPU by tsat_ilp_build
# (csrc/ilp.cu); rows are materialised on the host in the reference's
# dictionary form only when asked for.  The solver is scipy's HiGHS MILP
# (library code, like the reference's scipy LP relaxations).

INT_TOL = 1e-6
COST_TOL = 1e-9


class ILPModel:
    """Objective and constraints (1)-(3), plus (4)/(5) with cycle constraints
    (reference extract.py:163-195: same fields, names, order and values)."""

    def __init__(self, **kw):
        self._rows = kw.pop("rows", None)
        self._skel = kw.pop("skeleton", None)
        for k, v in kw.items():
            setattr(self, k, v)

    @property
    def rows(self) -> list:
        if self._rows is None:
            self._rows = _materialize_rows(self)
        return self._rows

    @property
    def num_vars(self) -> int:
        return len(self.var_names)

    @property
    def num_classes(self) -> int:
        return len(self.class_order)

    def pin(self, node_id: int, value: int) -> None:
        idx = self.x_of_node[node_id]
        self.lb[idx] = self.ub[idx] = float(value)


def _ilp_skeleton(eg: EGraph, filt) -> dict:
    eg.set_filter(filt)
    lib = _lib.load()
    sizes = np.zeros(4, np.uint32)
    _lib.check(eg._h, lib.tsat_ilp_build(eg._h, _lib.ptr(sizes, C.c_uint32)))
    nr, nx, nl, npk = (int(x) for x in sizes)
    out = {"classes": np.zeros(max(nr, 1), np.uint32), "nodes": np.zeros(max(nx, 1), np.uint32),
           "live_off": np.zeros(nr + 1, np.uint32), "live": np.zeros(max(nl, 1), np.uint32),
           "pick_off": np.zeros(nl + 1, np.uint32), "pick_child": np.zeros(max(npk, 1), np.uint32)}
    _lib.check(eg._h, lib.tsat_ilp_download(
        eg._h, *(_lib.ptr(out[k], C.c_uint32) for k in
                 ("classes", "nodes", "live_off", "live", "pick_off", "pick_child"))))
    out["classes"] = out["classes"][:nr]
    out["nodes"] = out["nodes"][:nx]
    out["live"] = out["live"][:nl]
    out["pick_child"] = out["pick_child"][:npk]
    return out


def reachable_classes(eg: EGraph, filt, root: int) -> list:
    """Classes reachable from the root through live nodes, root first, then
    ascending (extract.py:198-217); BFS on the GPU."""
    if eg.find(root) != eg.find(eg.root):
        raise ValueError("the device BFS starts at the e-graph root")
    return [int(c) for c in _ilp_skeleton(eg, {int(x) for x in filt})["classes"]]


def build_ilp(eg: EGraph, costs: Mapping, filt: Iterable[int] = (), with_cycle: bool = False,
              topo: str = "real") -> ILPModel:
    """build_ilp (extract.py:220-322); unreachable classes pruned."""
    if eg.root is None:
        raise ExtractionError("e-graph has no root")
    if topo not in ("real", "int"):
        raise ValueError("topo must be 'real' or 'int'")
    filt = {int(x) for x in filt}
    sk = _ilp_skeleton(eg, filt)
    classes = [int(c) for c in sk["classes"]]
    m_count = len(classes)
    epsilon = 1.0 / (2 * m_count)
    big_a = float(m_count) if topo == "int" else 2.0
    nodes = sk["nodes"]
    node_list = nodes.tolist()
    x_of_node = {nid: i for i, nid in enumerate(node_list)}
    var_names = [f"x_{nid}" for nid in node_list]
    if isinstance(costs, CostVector):
        objective = costs.gather(nodes).tolist() if len(nodes) else []
    else:
        objective = [float(costs[nid]) for nid in node_list]
    pinned = {nid for nid in node_list if nid in filt}
    lb = [0.0] * len(node_list)
    ub = [0.0 if nid in pinned else 1.0 for nid in node_list]
    binary_idx = list(range(len(node_list)))
    t_of_class: dict = {}
    integer_idx: list = []
    if with_cycle:
        t_max = float(m_count - 1) if topo == "int" else 1.0
        for i, cid in enumerate(classes):
            t_of_class[cid] = len(var_names)
            var_names.append(f"t_{i}")
            objective.append(0.0)
            lb.append(0.0)
            ub.append(t_max)
            if topo == "int":
                integer_idx.append(t_of_class[cid])
    sk["live_x"] = np.searchsorted(nodes, sk["live"]).astype(np.int64)
    return ILPModel(
        var_names=var_names, objective=objective, lb=lb, ub=ub, binary_idx=binary_idx,
        integer_idx=integer_idx, x_of_node=x_of_node, node_of_x={v: k for k, v in x_of_node.items()},
        t_of_class=t_of_class, class_order=classes, root_class=classes[0],
        costs=costs if isinstance(costs, CostVector) else dict(costs), pinned=pinned,
        with_cycle=with_cycle, topo=topo, epsilon=epsilon, big_a=big_a, skeleton=sk)


def _materialize_rows(model: ILPModel) -> list:
    """Rows in the reference order (extract.py:280-306): root row, then per
    reachable class and live member, its pick rows (one per distinct child
    class, ascending id), then its topological rows."""
    sk = model._skel
    live_off = sk["live_off"].tolist()
    live = sk["live"].tolist()
    live_x = sk["live_x"].tolist()
    pick_off = sk["pick_off"].tolist()
    pick_child = sk["pick_child"].tolist()
    per_class = [live_x[live_off[k]:live_off[k + 1]] for k in range(len(model.class_order))]
    t_idx = [model.t_of_class[c] for c in model.class_order] if model.with_cycle else None
    rhs_topo = model.big_a - (1.0 if model.topo == "int" else model.epsilon)
    rows = [("root", {x: 1.0 for x in per_class[0]}, "=", 1.0)]
    for k in range(len(model.class_order)):
        for t in range(live_off[k], live_off[k + 1]):
            nid, xn = live[t], live_x[t]
            children = pick_child[pick_off[t]:pick_off[t + 1]]
            for m in children:
                coeffs = {xn: 1.0}
                for xj in per_class[m]:
                    coeffs[xj] = coeffs.get(xj, 0.0) - 1.0
                rows.append((f"pick_{nid}_c{m}", coeffs, "<=", 0.0))
            if model.with_cycle:
                for m in children:
                    coeffs = {xn: model.big_a}
                    ti, tm = t_idx[k], t_idx[m]
                    if ti != tm:
                        coeffs[tm] = coeffs.get(tm, 0.0) + 1.0
                        coeffs[ti] = coeffs.get(ti, 0.0) - 1.0
                    rows.append((f"topo_{nid}_c{m}", coeffs, "<=", rhs_topo))
    return rows


# ---------------------------------------------------------------- LP export


def _fmt(x: float) -> str:
    return f"{x:.12g}"


def _fmt_terms(coeffs: Mapping, names) -> str:
    parts = []
    for idx in sorted(coeffs):
        c = coeffs[idx]
        if c == 0:
            continue
        mag = _fmt(abs(c))
        if parts:
            parts.append(f"{'-' if c < 0 else '+'} {mag} {names[idx]}")
        else:
            parts.append(f"{'- ' if c < 0 else ''}{mag} {names[idx]}")
    return " ".join(parts) if parts else f"0 {names[0]}"


def export_lp(model: ILPModel) -> str:
    """CPLEX LP text, byte-identical to the reference's export_lp (extract.py:350-375)."""
    names = model.var_names
    cyc = "none" if not model.with_cycle else model.topo
    out = [f"\\ tensorsat extraction model: classes={model.num_classes} vars={model.num_vars} cycle={cyc}",
           "Minimize", " obj: " + _fmt_terms(dict(enumerate(model.objective)), names), "Subject To"]
    out += [f" {name}: {_fmt_terms(co, names)} {sense} {_fmt(rhs)}" for name, co, sense, rhs in model.rows]
    out.append("Bounds")
    tset = set(model.t_of_class.values())
    for idx, name in enumerate(names):
        lo, hi = model.lb[idx], model.ub[idx]
        if idx in tset:
            out.append(f" {_fmt(lo)} <= {name} <= {_fmt(hi)}")
        elif lo == hi:
            out.append(f" {name} = {_fmt(lo)}")
    out.append("Binary")
    out += [f" {names[i]}" for i in model.binary_idx]
    if model.integer_idx:
        out.append("General")
        out += [f" {names[i]}" for i in model.integer_idx]
    out.append("End")
    return "\n".join(out) + "\n"


# ------------------------------------------------------------------ solver


def _lp_arrays(model: ILPModel):
    from scipy import sparse

    n = model.num_vars
    mats = {}
    for sense in ("<=", "="):
        ri, ci, data, rhs = [], [], [], []
        for name, co, s_, b in model.rows:
            if s_ != sense:
                continue
            k = len(rhs)
            rhs.append(b)
            for idx, c in co.items():
                if c != 0:
                    ri.append(k)
                    ci.append(idx)
                    data.append(c)
        mats[sense] = (sparse.csr_matrix((data, (ri, ci)), shape=(len(rhs), n)), np.array(rhs)) if rhs else (None, None)
    return np.array(model.objective), mats["<="][0], mats["<="][1], mats["="][0], mats["="][1]


def solve_ilp(model: ILPModel, eg: EGraph, time_limit_s: float = 60.0) -> ExtractionResult:
    """Exact MILP solve of the model (scipy HiGHS branch-and-cut; the
    reference runs its own best-first branch-and-bound over scipy LP
    relaxations, extract.py:406-514).  Same optimum; among equal-cost optima
    the chosen selection may differ."""
    from scipy.optimize import Bounds, LinearConstraint, milp

    from .errors import InfeasibleModel, SolveTimeout

    t0 = time.perf_counter()
    if time_limit_s <= 0:  # no budget: the reference's search loop never starts (extract.py:464, 516)
        raise SolveTimeout(f"no feasible incumbent within {time_limit_s}s")
    c, a_ub, b_ub, a_eq, b_eq = _lp_arrays(model)
    integ = np.zeros(model.num_vars)
    integ[model.binary_idx] = 1
    if model.integer_idx:
        integ[model.integer_idx] = 1
    cons = []
    if a_ub is not None:
        cons.append(LinearConstraint(a_ub, -np.inf, b_ub))
    if a_eq is not None:
        cons.append(LinearConstraint(a_eq, b_eq, b_eq))
    res = milp(c, constraints=cons, integrality=integ, bounds=Bounds(model.lb, model.ub),
               options={"time_limit": float(time_limit_s)})
    stats = SolverStats(nodes_explored=int(getattr(res, "mip_node_count", 0) or 0), lp_solves=0,
                        time_s=time.perf_counter() - t0, optimal=res.status == 0)
    if res.x is None:
        if res.status == 1:
            raise SolveTimeout(f"no feasible incumbent within {time_limit_s}s")
        if res.status == 2:
            raise InfeasibleModel("no selection satisfies the constraints")
        raise ExtractionError(f"MILP solve failed: {res.message}")
    x = res.x
    selected = [model.node_of_x[i] for i in model.binary_idx if x[i] > 0.5]
    stats.objective = float(sum(model.objective[i] for i in model.binary_idx if x[i] > 0.5))
    return _result_from_nodes(model, eg, selected, stats)


def _find_many(eg: EGraph, ids) -> list:
    ids = np.asarray(list(ids), np.uint32)
    out = np.zeros(max(len(ids), 1), np.uint32)
    _lib.check(eg._h, _lib.load().tsat_find_batch(eg._h, len(ids), _lib.ptr(ids, C.c_uint32),
                                                  _lib.ptr(out, C.c_uint32)))
    return out[: len(ids)].tolist()


def _result_from_nodes(model: ILPModel, eg: EGraph, selected, stats: SolverStats) -> ExtractionResult:
    """extract.py:517-541: min node per selected class, restricted to the
    classes reached from the root, pinned / acyclicity checks."""
    from .errors import CyclicSelection

    chosen: dict = {}
    for nid, cid in zip(selected, _find_many(eg, selected)):
        chosen[cid] = min(chosen.get(cid, nid), nid)
    kids = {nid: ch for nid, (_, ch) in _selected_nodes(eg, chosen.values()).items()} if chosen else {}
    all_kids = sorted({k for ch in kids.values() for k in ch})
    canon = dict(zip(all_kids, _find_many(eg, all_kids))) if all_kids else {}
    root = eg.find(model.root_class)
    selection: dict = {}
    stack = [root]
    while stack:
        cid = stack.pop()
        if cid in selection:
            continue
        if cid not in chosen:
            raise ReconstructError(f"no selected node covers e-class c{cid}")
        selection[cid] = chosen[cid]
        stack.extend(canon[k] for k in kids[chosen[cid]])
    for cid, nid in selection.items():
        if nid in model.pinned:
            raise ExtractionError(f"filter-listed node n{nid} selected")
    state: dict = {}

    def acyclic(c0) -> bool:  # iterative DFS over the selection
        todo = [(c0, 0)]
        while todo:
            c, i = todo.pop()
            ch = kids[selection[c]]
            if i == 0:
                if state.get(c) == 2:
                    continue
                if state.get(c) == 1:
                    return False
                state[c] = 1
            if i < len(ch):
                todo.append((c, i + 1))
                d = canon[ch[i]]
                if state.get(d) == 1:
                    return False
                if state.get(d) != 2:
                    todo.append((d, 0))
            else:
                state[c] = 2
        return True

    if not all(acyclic(c) for c in selection):
        raise CyclicSelection("extracted selection contains a cycle"
                              + ("" if model.with_cycle else " (filter list was insufficient)"))
    return ExtractionResult(selection, selection_cost(model.costs, selection), stats=stats,
                            optimal=stats.optimal)


def parse_solution(model: ILPModel, eg: EGraph, text: str) -> ExtractionResult:
    """Import an external solver's ``variable = value`` lines (extract.py:544-578)."""
    from .errors import GraphParseError

    values: dict = {}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" in line:
            name, _, val = line.partition("=")
        else:
            parts = line.split()
            if len(parts) != 2:
                raise GraphParseError(f"bad solution line {line!r}", line=lineno)
            name, val = parts
        try:
            values[name.strip()] = float(val)
        except ValueError:
            raise GraphParseError(f"bad value in {line!r}", line=lineno) from None
    index = {name: i for i, name in enumerate(model.var_names)}
    unknown = sorted(set(values) - set(index))
    if unknown:
        raise GraphParseError(f"unknown variables {unknown[:3]}")
    binaries = set(model.binary_idx)
    selected = [model.node_of_x[index[n]] for n, v in values.items() if index[n] in binaries and v > 0.5]
    stats = SolverStats(optimal=False)
    stats.objective = sum(model.costs[n] for n in selected)
    return _result_from_nodes(model, eg, selected, stats)
