"""GPU-resident e-graph (the reference's ``EGraph`` API on top of libtsat).

Every mutation and query runs on the device through the C-ABI; the Python
object only keeps the atom intern table and a lazily downloaded read-only
view (``nodes`` / ``classes``) for callers that walk the graph, e.g.
``reconstruct`` or tests.  Interface: reference pkg/src/tensorsat/egraph.py
:42-364 (UnionFind semantics: class id = smallest node id; node ids are the
global insertion counter; ``dump`` byte-identical).
"""

from __future__ import annotations

import functools

import ctypes as C
import itertools
from dataclasses import dataclass
from typing import Any, Iterable, Iterator, Mapping, Optional, Protocol

import numpy as np

from . import _lib
from .errors import ShapeMismatch
from .rules import Match, canonicalize
from .sexpr import App, Atom, Term, Var, variables

NONE = 0xFFFFFFFF

VAL_DTYPE = np.dtype(
    [("kind", "i1"), ("r0", "i1"), ("r1", "i1"), ("n0", "i1"), ("n1", "i1"), ("pad", "i1", 3),
     ("iv", "<i8"), ("d0", "<i8", 4), ("d1", "<i8", 4), ("o0", "<u4", 6), ("o1", "<u4", 6)]
)
_ATOM_ROWS: dict = {}  # encoded atom tables by atom sequence (_flush_atoms)
TREE_DTYPE = np.dtype([("npos", "<i4"), ("pad", "<i4"), ("pos", "<i8", 5), ("kid", "<u4", 6), ("pad2", "<u4", 14)])
assert VAL_DTYPE.itemsize == 128 and TREE_DTYPE.itemsize == 128


@dataclass
class ENode:
    id: int
    op: Atom
    children: tuple


@dataclass
class EClass:
    id: int
    node_ids: set
    analysis: Any = None


@functools.lru_cache(maxsize=None, typed=True)
def _atom_info(a: Atom):
    """(kind, ival, opcode, ndims, dims, nident, idims) for the device atom table;
    string parsing mirrors tensor_lang.parse_dims / parse_identifier."""
    from .tensor_lang import OP_CODES

    def dims_of(s):
        try:
            d = tuple(int(p) for p in s.split("_"))
        except ValueError:
            return -1, (0, 0, 0, 0)
        return len(d), tuple(list(d[:4]) + [0] * (4 - min(4, len(d))))

    if isinstance(a, bool) or not isinstance(a, (int, str)):
        raise TypeError(f"atoms must be int or str, got {a!r}")
    if isinstance(a, int):
        if not -(1 << 63) <= a < (1 << 63):
            raise ValueError(f"integer atom {a} does not fit the device's int64")
        return 0, a, -1, -1, (0, 0, 0, 0), -1, (0, 0, 0, 0)
    nd, dims = dims_of(a)
    ni, idims = -1, (0, 0, 0, 0)
    if "@" in a:
        name, _, ds = a.rpartition("@")
        if name:
            ni, idims = dims_of(ds)
    for d in list(dims) + list(idims):
        if not -(1 << 63) <= d < (1 << 63):
            raise ValueError(f"dimension in {a!r} does not fit int64")
    return 1, 0, OP_CODES.get(a, -1), nd, dims, ni, idims


class _View:
    """Host copy of the device SoA, valid until the next mutation."""

    def __init__(self, eg: "EGraph"):
        n, live, nk, root, _ = eg._sizes()
        self.n = n
        self.op = np.zeros(n, np.uint32)
        self.koff = np.zeros(n + 1, np.uint32)
        self.kids = np.zeros(max(nk, 1), np.uint32)
        self.cls = np.zeros(n, np.uint32)
        self.flags = np.zeros(n, np.uint8)
        lib = _lib.load()
        _lib.check(eg._h, lib.tsat_download(
            eg._h, _lib.ptr(self.op, C.c_uint32), _lib.ptr(self.koff, C.c_uint32),
            _lib.ptr(self.kids, C.c_uint32), _lib.ptr(self.cls, C.c_uint32), _lib.ptr(self.flags, C.c_uint8)))
        self.alive = (self.flags & 1).astype(bool)
        self.filtered = (self.flags & 2).astype(bool)
        self.atoms = eg._atom_list
        self._nodes = None
        self._classes = None
        self.values = None
        if eg.analysis is not None:
            self.values = np.zeros(n, VAL_DTYPE)
            nt = C.c_uint32()
            _lib.check(eg._h, lib.tsat_download_values(eg._h, None, 0, None, 0, C.byref(nt)))
            self.trees = np.zeros(max(nt.value, 1), TREE_DTYPE)
            _lib.check(eg._h, lib.tsat_download_values(
                eg._h, self.values.ctypes.data_as(C.c_void_p), self.values.nbytes,
                self.trees.ctypes.data_as(C.c_void_p), self.trees.nbytes, C.byref(nt)))
            self._tree_cache = {}

    def node(self, nid: int) -> ENode:
        a, b = int(self.koff[nid]), int(self.koff[nid + 1])
        return ENode(nid, self.atoms[int(self.op[nid])], tuple(int(x) for x in self.kids[a:b]))

    @property
    def nodes(self) -> dict:
        if self._nodes is None:
            self._nodes = {int(i): self.node(int(i)) for i in np.nonzero(self.alive)[0]}
        return self._nodes

    @property
    def classes(self) -> dict:
        if self._classes is None:
            out: dict = {}
            for i in np.nonzero(self.alive)[0]:
                c = int(self.cls[i])
                ec = out.get(c)
                if ec is None:
                    ec = out[c] = EClass(c, set(), None)
                ec.node_ids.add(int(i))
            if self.values is not None:
                for c, ec in out.items():
                    ec.analysis = self.value(c)
            self._classes = dict(sorted(out.items()))
        return self._classes

    def _tree(self, tid: int):
        if tid == 0x0FFFFFFF:
            return None
        t = self._tree_cache.get(tid)
        if t is None:
            rec = self.trees[tid]
            npos = int(rec["npos"])
            t = (tuple(int(x) for x in rec["pos"][:npos]),
                 tuple(self._tree(int(k)) for k in rec["kid"][: npos + 1]))
            self._tree_cache[tid] = t
        return t

    def _origins(self, arr, n):
        return frozenset((int(e) >> 28, self._tree(int(e) & 0x0FFFFFFF)) for e in arr[:n])

    def value(self, c: int):
        from .tensor_lang import Value

        v = self.values[c]
        k = int(v["kind"])
        if k == 1:
            return Value.of_int(int(v["iv"]))
        if k == 2:
            return Value.of_str(self.atoms[int(v["iv"])])
        if k == 3:
            return Value.of_tensor(tuple(int(x) for x in v["d0"][: v["r0"]]),
                                   self._origins(v["o0"], int(v["n0"])))
        if k == 4:
            return Value.of_pair(
                tuple(int(x) for x in v["d0"][: v["r0"]]), tuple(int(x) for x in v["d1"][: v["r1"]]),
                self._origins(v["o0"], int(v["n0"])), self._origins(v["o1"], int(v["n1"])))
        return None


class Analysis(Protocol):
    """Language client of the e-graph (reference egraph.py:28-39).  The device
    engine implements the tensor analysis natively (``TensorAnalysis``) or
    none; the protocol is kept for type annotations of client code."""

    def make(self, op: Atom, child_values: list) -> Any: ...

    def merge(self, a: Any, b: Any) -> Any: ...


class UnionFind:
    """Host union-find with the reference's contract (egraph.py:42-71): the
    representative is the SMALLEST id.  The engine's own union-find lives on
    the device (csrc/common.cuh uf_find / uf_union_min); this class serves
    client code and tests that use the reference type directly."""

    __slots__ = ("_parent",)

    def __init__(self) -> None:
        self._parent: dict = {}

    def make(self, x: int) -> None:
        self._parent[x] = x

    def find(self, x: int) -> int:
        p = self._parent
        while p[x] != x:  # path halving
            p[x] = p[p[x]]
            x = p[x]
        return x

    def union(self, a: int, b: int) -> int:
        ra, rb = self.find(a), self.find(b)
        if ra != rb:
            lo, hi = min(ra, rb), max(ra, rb)
            self._parent[hi] = lo
            return lo
        return ra

    def copy(self) -> "UnionFind":
        out = UnionFind()
        out._parent = self._parent.copy()
        return out


class EGraph:
    """Device-backed e-graph with the reference's public interface."""

    def __init__(self, analysis=None, device: int = 0):
        self.analysis = analysis
        self.device = device
        lib = _lib.load()
        h = C.c_void_p()
        st = lib.tsat_create(device, 0 if analysis is None else 1, C.byref(h))
        if st != 0:
            raise _lib.E.DeviceError(f"tsat_create failed with status {st} (is a CUDA device visible?)")
        self._h = h
        self._atoms: dict = {}
        self._atom_list: list = []
        self._sent = 0
        self._view: Optional[_View] = None
        self._filt_dev: Optional[frozenset] = frozenset()  # filter list known to be on the device

    def clone(self) -> "EGraph":
        """Independent copy (reference egraph.py:351-364): a second engine on
        the same device, filled by a device-to-device copy of the node table,
        union-find, analyses, cut trees and hashcons (tsat_copy_state)."""
        self._flush_atoms()
        other = EGraph(self.analysis, self.device)
        other._atoms = dict(self._atoms)
        other._atom_list = list(self._atom_list)
        other._sent = 0
        other._flush_atoms()
        _lib.check(other._h, _lib.load().tsat_copy_state(other._h, self._h))
        other._filt_dev = self._filt_dev
        return other

    def eval_patterns(self, terms, substs) -> list:
        """Device shape inference of each term under its substitution
        (rules.eval_pattern, reference rules.py:126-138): one program per term
        in the add_term format, evaluated by k_eval_terms without inserting."""
        from .errors import MissingSplitOrigin

        progs, env, env_off = [], [], []
        for term, sub in zip(terms, substs):
            slots: dict = {}
            env_off.append(len(env))

            def slot_of(name, slots=slots, sub=sub):
                if name not in slots:
                    slots[name] = len(slots)
                    env.append(int(sub[name]))
                return slots[name]

            progs.append(compile_term(term, self._atom, slot_of))
        self._flush_atoms()
        instr = np.array([x for prog in progs for ins in prog for x in ins] or [0], np.int32)
        lens = np.array([len(p) for p in progs], np.int32)
        envv = np.array(env or [0], np.uint32)
        offs = np.array(env_off or [0], np.uint32)
        vals = np.zeros(max(len(progs), 1), VAL_DTYPE)
        status = np.zeros(max(len(progs), 1), np.int32)
        lib = _lib.load()
        _lib.check(self._h, lib.tsat_eval_terms(
            self._h, int(lens.sum()), _lib.ptr(instr, C.c_int32), len(progs), _lib.ptr(lens, C.c_int32), len(env),
            _lib.ptr(envv, C.c_uint32), _lib.ptr(offs, C.c_uint32), vals.ctypes.data_as(C.c_void_p),
            _lib.ptr(status, C.c_int32)))
        for i, st in enumerate(status[: len(progs)]):
            if st == 2:
                raise MissingSplitOrigin(f"split of {terms[i]} has no recorded origin on its axis")
            if st != 0:
                raise ShapeMismatch(f"pattern {terms[i]} does not shape-check")
        nt = C.c_uint32()
        _lib.check(self._h, lib.tsat_download_values(self._h, None, 0, None, 0, C.byref(nt)))
        view = _View.__new__(_View)
        view.values = vals
        view.trees = np.zeros(max(nt.value, 1), TREE_DTYPE)
        _lib.check(self._h, lib.tsat_download_values(self._h, None, 0, view.trees.ctypes.data_as(C.c_void_p),
                                                       view.trees.nbytes, C.byref(nt)))
        view.atoms = self._atom_list
        view._tree_cache = {}
        return [view.value(i) for i in range(len(progs))]

    @property
    def reach_budget(self) -> None:
        raise AttributeError("write-only")

    @reach_budget.setter
    def reach_budget(self, nbytes: int) -> None:
        """Bytes the efficient pre-filter may spend on the C x C descendants
        bitset (reference cycles.py:70-148) before it answers reaches() from
        the peel levels + a pruned search; 0 forces the latter."""
        _lib.check(self._h, _lib.load().tsat_set_reach_budget(self._h, int(nbytes)))

    @property
    def reach_mode(self) -> int:
        out = C.c_int32()
        _lib.check(self._h, _lib.load().tsat_reach_mode(self._h, C.byref(out)))
        return out.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.tsat_destroy(h)
            self._h = None

    # ---------------------------------------------------------------- atoms
    def _atom(self, a: Atom) -> int:
        key = (type(a) is int, a)
        i = self._atoms.get(key)
        if i is None:
            _atom_info(a)  # validate early
            i = self._atoms[key] = len(self._atom_list)
            self._atom_list.append(a)
        return i

    def _flush_atoms(self) -> None:
        n = len(self._atom_list)
        if n == self._sent:
            return
        key = tuple((type(a) is int, a) for a in self._atom_list)
        rows = _ATOM_ROWS.get(key)
        if rows is None:  # the same atom sequence (same graph / rules) reuses its encoded table
            info = [_atom_info(a) for a in self._atom_list]
            names = [str(a).encode() for a in self._atom_list]
            off = np.zeros(n + 1, np.int64)
            off[1:] = np.cumsum([len(b) for b in names])
            rows = (np.array([x[0] for x in info], np.int32), np.array([x[1] for x in info], np.int64),
                    np.array([x[2] for x in info], np.int32), np.array([x[3] for x in info], np.int32),
                    np.array([x[4] for x in info], np.int64).reshape(-1), np.array([x[5] for x in info], np.int32),
                    np.array([x[6] for x in info], np.int64).reshape(-1), b"".join(names) + b"\0", off)
            if len(_ATOM_ROWS) > 64:
                _ATOM_ROWS.clear()
            _ATOM_ROWS[key] = rows
        kind, ival, opc, nd, dims, ni, idims, blob, off = rows
        lib = _lib.load()
        _lib.check(self._h, lib.tsat_set_atoms(
            self._h, n, _lib.ptr(kind, C.c_int32), _lib.ptr(ival, C.c_int64), _lib.ptr(opc, C.c_int32),
            _lib.ptr(nd, C.c_int32), _lib.ptr(dims, C.c_int64), _lib.ptr(ni, C.c_int32),
            _lib.ptr(idims, C.c_int64), blob, _lib.ptr(off, C.c_int64)))
        self._sent = n

    def _touch(self) -> None:
        self._view = None

    # ---------------------------------------------------------------- sizes
    def _sizes(self):
        v = [C.c_uint32() for _ in range(5)]
        _lib.check(self._h, _lib.load().tsat_query_sizes(self._h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    @property
    def num_nodes(self) -> int:
        return self._sizes()[1]

    @property
    def num_classes(self) -> int:
        out = C.c_uint32()
        _lib.check(self._h, _lib.load().tsat_num_classes(self._h, C.byref(out)))
        return out.value

    def _alive_flags(self) -> np.ndarray:
        n = self._sizes()[0]
        fl = np.zeros(max(n, 1), np.uint8)
        _lib.check(self._h, _lib.load().tsat_download_flags(self._h, _lib.ptr(fl, C.c_uint8)))
        return (fl[:n] & 1).astype(bool)

    @property
    def allocated_nodes(self) -> int:
        return self._sizes()[0]

    @property
    def root(self) -> Optional[int]:
        r = self._sizes()[3]
        return None if r == NONE else r

    @root.setter
    def root(self, cid: Optional[int]) -> None:
        _lib.check(self._h, _lib.load().tsat_set_root(self._h, NONE if cid is None else int(cid)))

    @property
    def view(self) -> _View:
        if self._view is None:
            self._view = _View(self)
        return self._view

    @property
    def nodes(self) -> dict:
        return self.view.nodes

    @property
    def classes(self) -> dict:
        return self.view.classes

    # ---------------------------------------------------------------- construction
    def _load_initial(self, ops, kids, root) -> None:
        atom = self._atom
        op_ids = np.fromiter((atom(o) for o in ops), np.uint32, len(ops))
        self._flush_atoms()
        koff = np.zeros(len(ops) + 1, np.uint32)
        koff[1:] = np.cumsum(np.fromiter(map(len, kids), np.uint32, len(kids)))
        flat = np.fromiter(itertools.chain.from_iterable(kids), np.uint32, int(koff[-1])) if koff[-1] else \
            np.zeros(1, np.uint32)
        _lib.check(self._h, _lib.load().tsat_load_egraph(
            self._h, len(ops), _lib.ptr(op_ids, C.c_uint32), _lib.ptr(koff, C.c_uint32),
            _lib.ptr(flat, C.c_uint32), root))
        self._touch()

    def _run_terms(self, programs, env_list) -> list:
        instr = np.array([x for prog in programs for ins in prog for x in ins] or [0], np.int32)
        lens = np.array([len(p) for p in programs], np.int32)
        env = np.array(env_list or [0], np.uint32)
        self._flush_atoms()
        out = np.zeros(len(programs), np.uint32)
        _lib.check(self._h, _lib.load().tsat_add_terms(
            self._h, int(sum(lens)), _lib.ptr(instr, C.c_int32), len(programs), _lib.ptr(lens, C.c_int32),
            len(env_list), _lib.ptr(env, C.c_uint32), _lib.ptr(out, C.c_uint32)))
        self._touch()
        return [int(x) for x in out]

    def add_enode(self, op: Atom, children: Iterable[int] = ()) -> int:
        ch = [int(c) for c in children]
        prog = [(0, i, 0, 0) for i in range(len(ch))] + [(1, len(ch), self._atom(op), 1)]
        return self._run_terms([prog], ch)[0]

    def add_term(self, term: Term, env: Optional[Mapping[str, int]] = None) -> int:
        slots: dict = {}
        envl: list = []
        prog = compile_term(term, self._atom, lambda v: _slot(v, env, slots, envl))
        return self._run_terms([prog], envl)[0]

    def union(self, a: int, b: int) -> int:
        out = C.c_uint32()
        _lib.check(self._h, _lib.load().tsat_union(self._h, int(a), int(b), C.byref(out)))
        self._touch()
        return out.value

    def rebuild(self) -> None:
        _lib.check(self._h, _lib.load().tsat_rebuild(self._h))
        self._touch()

    # ---------------------------------------------------------------- queries
    def find(self, cid: int) -> int:
        v = self._view
        if v is not None and 0 <= cid < v.n:
            return int(v.cls[cid])
        out = C.c_uint32()
        _lib.check(self._h, _lib.load().tsat_find(self._h, int(cid), C.byref(out)))
        return out.value

    def class_of(self, nid: int) -> int:
        return self.find(nid)

    def eclass(self, cid: int) -> EClass:
        return self.classes[self.find(cid)]

    def class_ids(self) -> list:
        return list(self.classes)

    def iter_nodes(self) -> Iterator[ENode]:
        nodes = self.nodes
        for nid in sorted(nodes):
            yield nodes[nid]

    def node_children(self, nid: int) -> tuple:
        return tuple(self.find(c) for c in self.nodes[nid].children)

    def dump(self) -> str:
        n = C.c_int64()
        lib = _lib.load()
        _lib.check(self._h, lib.tsat_dump(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _lib.check(self._h, lib.tsat_dump(self._h, buf, n.value + 1, C.byref(n)))
        return buf.raw[: n.value].decode()

    def set_filter(self, filt: Iterable[int]) -> None:
        """Replace the device filter list (every call taking ``filt`` uploads it)."""
        # the common call passes back the set saturate() returned: compare
        # before converting element by element
        want = filt if isinstance(filt, frozenset) else frozenset(filt)
        if self._filt_dev is not None and want == self._filt_dev:
            return
        want = frozenset(int(x) for x in want)
        if self._filt_dev is not None and want == self._filt_dev:
            return
        n_alloc = self._sizes()[0]
        lib = _lib.load()
        _lib.check(self._h, lib.tsat_set_filter(self._h, 0, None, 2))
        real = sorted({int(x) for x in filt if 0 <= int(x) < n_alloc})
        if real:
            arr = np.array(real, np.uint32)
            _lib.check(self._h, lib.tsat_set_filter(self._h, len(arr), _lib.ptr(arr, C.c_uint32), 1))
        self._filt_dev = frozenset(real)
        self._touch()

    def get_filter(self) -> list:
        lib = _lib.load()
        n = C.c_int64()
        cap = max(self._sizes()[0], 1)  # upper bound: one device compaction, no retry
        while True:
            out = np.empty(cap, np.uint32)
            _lib.check(self._h, lib.tsat_get_filter(self._h, _lib.ptr(out, C.c_uint32), cap, C.byref(n)))
            if n.value <= cap:
                return out[: n.value].tolist()
            cap = int(n.value)

    def ematch(self, pattern: Term, filt=frozenset()) -> list:
        """All matches of ``pattern`` (egraph.py:248-262), computed on the GPU."""
        self.set_filter(filt)
        if isinstance(pattern, Var):
            v = self.view
            out = []
            for c, ec in v.classes.items():
                if any(not v.filtered[n] for n in ec.node_ids):
                    out.append(Match(c, ((pattern.name, c),)))
            return out
        cp = canonicalize(pattern)
        blob, _ = compile_ruleset(self, [], extra_patterns=[cp.pattern])
        lib = _lib.load()
        _lib.check(self._h, lib.tsat_load_rules(self._h, len(blob), _lib.ptr(blob, C.c_int64)))
        n = C.c_int64()
        nb = C.c_int32()
        _lib.check(self._h, lib.tsat_ematch(self._h, 0, None, None, 0, C.byref(n), C.byref(nb)))
        cls = np.zeros(max(n.value, 1), np.uint32)
        bind = np.zeros(max(n.value * nb.value, 1), np.uint32)
        _lib.check(self._h, lib.tsat_ematch(self._h, 0, _lib.ptr(cls, C.c_uint32), _lib.ptr(bind, C.c_uint32),
                                            len(cls), C.byref(n), C.byref(nb)))
        names = sorted(f"v{i}" for i in range(nb.value))
        back = {c: o for o, c in cp.rename}
        out = []
        for r in range(n.value):
            b = bind[r * nb.value:(r + 1) * nb.value]
            out.append(Match(int(cls[r]), tuple(sorted((back[names[k]], int(b[k])) for k in range(nb.value)))))
        return out

    def represented_terms(self, cid: int, depth_limit: int, filt=frozenset()) -> set:
        """Ground terms of a class up to a depth (host walk over the downloaded view)."""
        v = self.view
        memo: dict = {}

        def go(c: int, d: int) -> set:
            c = int(v.cls[c])
            if d <= 0:
                return set()
            key = (c, d)
            if key in memo:
                return memo[key]
            memo[key] = set()
            out: set = set()
            for nid in sorted(v.classes[c].node_ids):
                if nid in filt:
                    continue
                nd = v.node(nid)
                if not nd.children:
                    out.add(App(nd.op))
                    continue
                if d == 1:
                    continue
                combos = [()]
                for ch in nd.children:
                    terms = go(ch, d - 1)
                    combos = [p + (t,) for p in combos for t in terms]
                    if not combos:
                        break
                for args in combos:
                    out.add(App(nd.op, args))
            memo[key] = out
            return out

        try:
            return go(cid, depth_limit)
        finally:
            go = None  # break the recursive closure's cycle (it references self)

    # ---------------------------------------------------------------- costs (cost.py)
    def _device_costs(self, model) -> "CostVector":
        lib = _lib.load()
        n = self._sizes()[0]
        out = None  # the vector stays on the device; CostVector downloads it lazily
        if model.mode == "table":
            keys = [k.encode() for k in model.table]
            off = np.zeros(len(keys) + 1, np.int64)
            off[1:] = np.cumsum([len(k) for k in keys])
            vals = np.array(list(model.table.values()) or [0.0], np.float64)
            blob = b"".join(keys) + b"\0"
            _lib.check(self._h, lib.tsat_costs(self._h, 1, 1 if model.strict else 0, len(keys), blob,
                                               _lib.ptr(off, C.c_int64), _lib.ptr(vals, C.c_double), None))
        else:
            _lib.check(self._h, lib.tsat_costs(self._h, 0, 0, 0, b"\0", None, None, None))
        return CostVector(self, None, None, n)


class CostVector(Mapping):
    """c_i per live node id (dict-like), backed by the device vector; the
    host copy and the live-node index are fetched lazily, and ``gather`` reads
    selected entries only (greedy_extract's total)."""

    def __init__(self, eg: EGraph, arr: Optional[np.ndarray], alive, n: Optional[int] = None):
        self._eg = eg
        self._arr = arr
        self._n = len(arr) if arr is not None else int(n)
        self._alive = alive
        self._ids = None

    @property
    def array(self) -> np.ndarray:
        if self._arr is None:
            out = np.zeros(max(self._n, 1), np.float64)
            _lib.check(self._eg._h, _lib.load().tsat_costs_gather(self._eg._h, self._n, None,
                                                                  _lib.ptr(out, C.c_double)))
            self._arr = out[: self._n]
        return self._arr

    def gather(self, ids) -> np.ndarray:
        ids = np.asarray(ids, np.uint32)
        if self._arr is not None:
            return self._arr[ids]
        out = np.zeros(max(len(ids), 1), np.float64)
        _lib.check(self._eg._h, _lib.load().tsat_costs_gather(self._eg._h, len(ids), _lib.ptr(ids, C.c_uint32),
                                                              _lib.ptr(out, C.c_double)))
        return out[: len(ids)]

    def _index(self):
        if self._alive is None:
            self._alive = self._eg._alive_flags()[: self._n]
        if self._ids is None:
            self._ids = np.nonzero(self._alive)[0]
        return self._ids

    def __getitem__(self, nid):
        nid = int(nid)
        if nid < 0 or nid >= self._n:
            raise KeyError(nid)
        self._index()
        if not self._alive[nid]:
            raise KeyError(nid)
        return float(self.array[nid])

    def __iter__(self):
        return (int(i) for i in self._index())

    def __len__(self):
        return len(self._index())


def _slot(v: str, env, slots: dict, envl: list) -> int:
    if env is None or v not in env:
        raise KeyError(f"unbound variable ?{v}")
    s = slots.get(v)
    if s is None:
        s = slots[v] = len(envl)
        envl.append(int(env[v]))
    return s


def compile_term(term: Term, atom_id, slot_of) -> list:
    """Post-order program (kind, arg, atom, depth) for add_term / targets."""
    prog: list = []

    def go(t) -> int:
        if isinstance(t, Var):
            prog.append((0, slot_of(t.name), 0, 0))
            return 0
        d = 0
        for a in t.args:
            d = max(d, go(a))
        prog.append((1, len(t.args), atom_id(t.op), d + 1))
        return d + 1

    go(term)
    go = None  # break the closure's self-reference (it holds atom_id, a bound method of the e-graph)
    return prog


def _compile_pattern(pat: Term, atom_id) -> list:
    """[napps, nvars, order..., (atom, nargs, child[8]) per app in pre-order]."""
    apps: list = []
    nvars = len(variables(pat))

    def go(t) -> int:
        idx = len(apps)
        apps.append(None)
        child = []
        for a in t.args:
            if isinstance(a, Var):
                child.append(-(int(a.name[1:]) + 1))
            else:
                child.append(go(a))
        if len(child) > 8:
            raise NotImplementedError("pattern arity > 8 is not supported on the device")
        apps[idx] = (atom_id(t.op), len(t.args), child + [0] * (8 - len(child)))
        return idx

    go(pat)
    go = None  # see compile_term
    names = sorted(f"v{i}" for i in range(nvars))
    out = [len(apps), nvars] + [int(n[1:]) for n in names]
    for atom, nargs, ch in apps:
        out += [atom, nargs] + ch
    return out


_RULESET_CACHE: dict = {}


def compile_ruleset(eg: EGraph, rules, extra_patterns=()):
    """Lower rules to the int64 blob of tsat_load_rules.  Returns (blob, pattern ids).

    The blob depends on the rules and on the atom ids the e-graph has interned
    so far; repeated explorations of the same graph with the same rule set
    (pooled engines) reuse the compiled blob and replay the atom interning."""
    atoms = getattr(eg, "_atom_list", None)
    try:
        key = None if atoms is None else ((type(eg).__name__,) + tuple((type(a) is int, a) for a in atoms),
                                          tuple(rules), tuple(extra_patterns))
        hit = None if key is None else _RULESET_CACHE.get(key)
    except TypeError:  # unhashable rule / pattern objects: compile every time
        key, hit = None, None
    if hit is not None:
        blob, pidx, new_atoms = hit
        for a in new_atoms:
            eg._atom(a)
        eg._flush_atoms()
        return blob, dict(pidx)
    n_before = len(atoms) if atoms is not None else 0
    blob, pidx = _compile_ruleset(eg, rules, extra_patterns)
    if key is not None:
        if len(_RULESET_CACHE) > 64:
            _RULESET_CACHE.clear()
        _RULESET_CACHE[key] = (blob, dict(pidx), list(eg._atom_list[n_before:]))
    return blob, pidx


def _compile_ruleset(eg: EGraph, rules, extra_patterns=()):
    pats: list = list(extra_patterns)
    pidx = {p: i for i, p in enumerate(pats)}
    rule_parts: list = []
    for r in rules:
        canon = r.canonical_sources
        slots: dict = {}
        for s in r.sources:
            for v in variables(s):
                slots.setdefault(v, len(slots))
        part = [len(r.sources), len(slots),
                1 if all(cp.pattern == canon[0].pattern for cp in canon[1:]) else 0]
        for cp in canon:
            if cp.pattern not in pidx:
                pidx[cp.pattern] = len(pats)
                pats.append(cp.pattern)
            back = {c: o for o, c in cp.rename}
            nv = len(cp.rename)
            names = sorted(f"v{i}" for i in range(nv))
            part += [pidx[cp.pattern], nv] + [slots[back[n]] for n in names]
        for t in r.targets:
            prog = compile_term(t, eg._atom, lambda v: slots[v])
            part.append(len(prog))
            for ins in prog:
                part += list(ins)
            leaves = variables(t)
            part += [len(leaves)] + [slots[v] for v in leaves]
        rule_parts.append(part)
    blob = [len(pats)]
    for p in pats:
        blob += _compile_pattern(p, eg._atom)
    blob.append(len(rules))
    for part in rule_parts:
        blob += part
    eg._flush_atoms()
    return np.array(blob, np.int64), pidx
