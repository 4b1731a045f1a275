"""Exploration entry points (reference: pkg/src/tensorsat/explorer.py:56-384).

``explore`` / ``saturate`` keep the reference signatures and result types; the
whole iteration loop -- e-matching, multi-pattern joins, shape and cycle
gates, application, rebuild, cycle post-processing -- runs on the GPU in
``tsat_saturate`` (csrc/explore.cu, csrc/wave.cu).
"""

from __future__ import annotations

import warnings

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _lib
from .egraph import EGraph, compile_ruleset
from .errors import AnalysisMergeError, TensorSatError
from .rules import Match, combined_subst
from .tensor_lang import TensorGraph, build_egraph

FILTER_MODES = ("none", "vanilla", "efficient")
_MODE_CODE = {"none": 0, "vanilla": 1, "efficient": 2}
_STOPS = ("iter-limit", "saturated", "node-limit", "timeout")


@dataclass
class ExploreLimits:
    n_max: int = 50000
    k_max: int = 15
    k_multi: int = 1
    time_limit_s: Optional[float] = None

    def __post_init__(self):
        if min(self.n_max, self.k_max, self.k_multi) < 0:
            raise ValueError("limits must be non-negative")
        if self.k_multi > self.k_max:
            raise ValueError("k_multi must be <= k_max")


@dataclass
class RuleStats:
    found: int = 0
    applied: int = 0
    applied_noop: int = 0
    skipped_self: int = 0
    skipped_compat: int = 0
    skipped_shape: int = 0
    skipped_cycle: int = 0


_RULE_FIELDS = ("found", "applied", "applied_noop", "skipped_self", "skipped_compat",
                "skipped_shape", "skipped_cycle")


@dataclass
class ExploreReport:
    iterations: int = 0
    stop_reason: str = ""
    enodes_per_iter: list = field(default_factory=list)
    alloc_per_iter: list = field(default_factory=list)
    eclasses_per_iter: list = field(default_factory=list)
    rules: dict = field(default_factory=dict)
    prefilter_checks: int = 0
    prefilter_rejects: int = 0
    postprocess_filtered: int = 0
    node_limit_overshoot: int = 0
    filter_size: int = 0
    time_s: float = 0.0

    @property
    def saturated(self) -> bool:
        return self.stop_reason == "saturated"

    def total(self, name: str) -> int:
        return sum(getattr(s, name) for s in self.rules.values())

    def to_stats(self) -> dict:
        out = {
            "explore.iterations": self.iterations,
            "explore.stop_reason": self.stop_reason,
            "explore.enodes_per_iter": ",".join(map(str, self.enodes_per_iter)),
            "explore.alloc_per_iter": ",".join(map(str, self.alloc_per_iter)),
            "explore.eclasses_per_iter": ",".join(map(str, self.eclasses_per_iter)),
            "explore.prefilter_checks": self.prefilter_checks,
            "explore.prefilter_rejects": self.prefilter_rejects,
            "explore.postprocess_filtered": self.postprocess_filtered,
            "explore.node_limit_overshoot": self.node_limit_overshoot,
            "explore.filter_size": self.filter_size,
            "explore.time_s": self.time_s,
        }
        for name, s in sorted(self.rules.items()):
            for f in _RULE_FIELDS:
                out[f"rule.{name}.{f}"] = getattr(s, f)
        return out


def iterate(
    eg: EGraph,
    rules: Sequence,
    iteration: int,
    limits: Optional[ExploreLimits] = None,
    filter_mode: str = "efficient",
    filt: Optional[set] = None,
    on_reject: Optional[Callable] = None,
    allow_self_pairs: bool = False,
):
    """One iteration of ``saturate`` as iteration number ``iteration`` of the
    caller's loop (multi-pattern rules active iff ``iteration < limits.k_multi``,
    explorer.py:338-352); ``tsat_iterate``.  Returns (filter list, ExploreReport)."""
    return saturate(eg, rules, limits, filter_mode, filt, on_reject, allow_self_pairs, _iteration=int(iteration))


def saturate(
    eg: EGraph,
    rules: Sequence,
    limits: Optional[ExploreLimits] = None,
    filter_mode: str = "efficient",
    filt: Optional[set] = None,
    on_reject: Optional[Callable] = None,
    allow_self_pairs: bool = False,
    _iteration: Optional[int] = None,
):
    """Iterate rules on ``eg`` (mutated in place) until saturation or a limit.
    Returns (filter list, ExploreReport); ``filt`` is updated in place.

    ``filter_mode="vanilla"`` checks each combo by applying it on a device
    checkpoint and running the cycle check from the root (cycles.py:248-254).
    ``on_reject(eg, filt, rule, matches)`` is the post-iteration variant of
    the reference hook (explorer.py:223-224): the device records every
    cycle-rejected combo (rule + snapshot Match per source, in rejection
    order) and the callbacks run after each iteration (the search is driven
    one iteration at a time), with the e-graph as that iteration left it; the
    live mid-iteration e-graph never leaves the GPU.  Recording keeps the
    wave path (rejected positions are logged on the device)."""
    limits = limits or ExploreLimits()
    if filter_mode not in FILTER_MODES:
        raise ValueError(f"filter_mode must be one of {FILTER_MODES}")
    if on_reject is not None and _iteration is None:
        return _saturate_per_iteration(eg, rules, limits, filter_mode, filt, on_reject, allow_self_pairs)
    filt = set() if filt is None else filt
    rules = list(rules)
    eg.set_filter(filt)
    blob, _ = compile_ruleset(eg, rules)
    lib = _lib.load()
    _lib.check(eg._h, lib.tsat_load_rules(eg._h, len(blob), _lib.ptr(blob, C.c_int64)))
    lim = _lib.Limits(limits.n_max, limits.k_max, limits.k_multi,
                      -1.0 if limits.time_limit_s is None else float(limits.time_limit_s))
    rep = _lib.Report()
    rs = np.zeros(max(len(rules), 1) * 7, np.int64)
    per = np.zeros(max(limits.k_max, 1) * 3, np.int64)
    if _iteration is not None and _iteration < 0:
        raise ValueError("iteration must be non-negative")
    if on_reject is not None:
        _lib.check(eg._h, lib.tsat_set_record_rejects(eg._h, 1))
    try:
        if _iteration is None:
            st = lib.tsat_saturate(eg._h, C.byref(lim), _MODE_CODE[filter_mode], 1 if allow_self_pairs else 0,
                                   C.byref(rep), _lib.ptr(rs, C.c_int64), _lib.ptr(per, C.c_int64))
        else:
            st = lib.tsat_iterate(eg._h, C.byref(lim), _MODE_CODE[filter_mode], 1 if allow_self_pairs else 0,
                                  _iteration, C.byref(rep), _lib.ptr(rs, C.c_int64), _lib.ptr(per, C.c_int64))
        _lib.check(eg._h, st)
    finally:
        eg._touch()
        if on_reject is not None:
            _lib.check(eg._h, lib.tsat_set_record_rejects(eg._h, 0))
    rejected = _rejected_combos(eg, rules) if on_reject is not None else []
    report = ExploreReport()
    for i, r in enumerate(rules):
        report.rules.setdefault(r.name, RuleStats(*[int(x) for x in rs[7 * i:7 * i + 7]]))
    it = int(rep.iterations)
    report.iterations = it
    report.stop_reason = _STOPS[rep.stop_reason]
    report.enodes_per_iter = [int(per[3 * i]) for i in range(it)]
    report.alloc_per_iter = [int(per[3 * i + 1]) for i in range(it)]
    report.eclasses_per_iter = [int(per[3 * i + 2]) for i in range(it)]
    report.prefilter_checks = int(rep.prefilter_checks)
    report.prefilter_rejects = int(rep.prefilter_rejects)
    report.postprocess_filtered = int(rep.postprocess_filtered)
    report.node_limit_overshoot = int(rep.node_limit_overshoot)
    report.time_s = float(rep.time_s)
    n_alloc = eg.allocated_nodes
    extra = {x for x in filt if not (0 <= int(x) < n_alloc)}
    filt.clear()
    dev = eg.get_filter()
    eg._filt_dev = frozenset(dev)
    filt.update(dev)
    filt.update(extra)
    report.filter_size = len(filt)
    if rejected:
        before = frozenset(filt)
        for rule, matches in rejected:
            on_reject(eg, filt, rule, matches)
        if frozenset(filt) != before:
            # the reference calls on_reject mid-iteration on the live e-graph
            # (explorer.py:222-224), so its filter edits steer the rest of that
            # iteration; here the callbacks run after the iteration and the
            # edits apply from the next one (API contract)
            warnings.warn("on_reject changed the filter list: the change takes effect from the next iteration "
                          "(callbacks run after each device iteration)", RuntimeWarning, stacklevel=2)
    return filt, report


def _saturate_per_iteration(eg, rules, limits, filter_mode, filt, on_reject, allow_self_pairs):
    """saturate() driven one iteration at a time (tsat_iterate), so on_reject
    sees each iteration's rejected combos right after that iteration, with the
    e-graph as the iteration left it (explorer.py:311-365 loop structure)."""
    import dataclasses
    import time

    t0 = time.perf_counter()
    filt = set() if filt is None else filt
    rules = list(rules)
    total = ExploreReport(stop_reason="iter-limit")
    for r in rules:
        total.rules.setdefault(r.name, RuleStats())
    for i in range(limits.k_max):
        lim = limits
        if limits.time_limit_s is not None:
            lim = dataclasses.replace(limits, time_limit_s=max(0.0, limits.time_limit_s - (time.perf_counter() - t0)))
        filt, rep = saturate(eg, rules, lim, filter_mode, filt, on_reject, allow_self_pairs, _iteration=i)
        total.iterations += rep.iterations
        total.enodes_per_iter += rep.enodes_per_iter
        total.alloc_per_iter += rep.alloc_per_iter
        total.eclasses_per_iter += rep.eclasses_per_iter
        for name, st in rep.rules.items():
            acc = total.rules.setdefault(name, RuleStats())
            for f in _RULE_FIELDS:
                setattr(acc, f, getattr(acc, f) + getattr(st, f))
        total.prefilter_checks += rep.prefilter_checks
        total.prefilter_rejects += rep.prefilter_rejects
        total.postprocess_filtered += rep.postprocess_filtered
        total.node_limit_overshoot = rep.node_limit_overshoot
        if rep.stop_reason != "iter-limit":
            total.stop_reason = rep.stop_reason
            break
    total.filter_size = len(filt)
    total.time_s = time.perf_counter() - t0
    return filt, total


def _rejected_combos(eg: EGraph, rules) -> list:
    """(rule, [Match per source]) for every cycle-rejected combo of the last
    tsat_saturate, in rejection order.  The device records the snapshot match
    rows; bindings are re-keyed by the rule's original variable names like
    run_rule's decanonicalize (explorer.py:231-233)."""
    lib = _lib.load()
    n = C.c_int64()
    _lib.check(eg._h, lib.tsat_rejects(eg._h, None, 0, C.byref(n)))
    buf = np.zeros(max(n.value, 1), np.uint32)
    _lib.check(eg._h, lib.tsat_rejects(eg._h, _lib.ptr(buf, C.c_uint32), len(buf), C.byref(n)))
    out, i = [], 0
    while i < n.value:
        rule = rules[int(buf[i])]
        nsrc = int(buf[i + 1])
        i += 2
        matches = []
        for t in range(nsrc):
            cls, nb = int(buf[i]), int(buf[i + 1])
            b = buf[i + 2:i + 2 + nb]
            i += 2 + nb
            names = sorted(f"v{k}" for k in range(nb))
            back = {c: o for o, c in rule.canonical_sources[t].rename}
            matches.append(Match(cls, tuple(sorted((back[names[k]], int(b[k])) for k in range(nb)))))
        out.append((rule, matches))
    return out


def _apply_combo(eg, rule, matches: Sequence[Match]) -> bool:
    """Instantiate each target under the combined substitution and union it
    with its matched class (reference explorer.py:146-163), through the
    device add_term / union; True iff nodes were allocated or a real merge
    happened.  The engine's own apply is the batched wave path (csrc/wave.cu);
    this is the single-combo form the reference API and vanilla_check use."""
    before = eg.allocated_nodes
    changed = False
    subst = combined_subst([m.subst for m in matches], eg)
    try:
        for tgt, m in zip(rule.targets, matches):
            new_cid = eg.add_term(tgt, subst)
            old_cid = eg.find(m.eclass)
            if eg.find(new_cid) != old_cid:
                eg.union(old_cid, new_cid)
                changed = True
    except AnalysisMergeError as e:
        raise AnalysisMergeError(f"unsound rule {rule.name!r}: {e}") from e
    return changed or eg.allocated_nodes > before


def explore(
    g: TensorGraph,
    rules: Sequence,
    limits: Optional[ExploreLimits] = None,
    filter_mode: str = "efficient",
    on_reject: Optional[Callable] = None,
    allow_self_pairs: bool = False,
    device: int = 0,
    shard_group=None,
):
    """End-to-end exploration of a single-rooted tensor graph on the GPU.
    ``shard_group``: a torch.distributed process group whose ranks (one per GPU)
    split e-matching by e-class range (shard.py); results are identical on
    every rank and to the single-GPU run."""
    if g.root is None:
        raise TensorSatError("graph must be single-rooted (run make_single_rooted)")
    eg, _ = build_egraph(g, device=device)
    if shard_group is not None:
        import torch.distributed as dist

        from .shard import attach_group, attach_host

        grp = None if shard_group is True else shard_group
        # NCCL over NVLink for an nccl group; a host (gloo) group exchanges
        # through host memory (several ranks may then share a GPU)
        (attach_host if dist.get_backend(grp) == "gloo" else attach_group)(eg, grp)
    filt, report = saturate(eg, rules, limits, filter_mode, on_reject=on_reject,
                            allow_self_pairs=allow_self_pairs)
    return eg, filt, report


def apply_multi_pattern(eg, multi_rules, filt=None, filter_mode="none", allow_self_pairs=False) -> int:
    """One multi-pattern pass (explorer.py:270-289)."""
    rules = [r for r in multi_rules if r.multi]
    filt, rep = saturate(eg, rules, ExploreLimits(n_max=1 << 62, k_max=1, k_multi=1), filter_mode,
                         filt=set() if filt is None else filt, allow_self_pairs=allow_self_pairs)
    return rep.total("applied")


def apply_single_patterns(eg, single_rules, filt=None, filter_mode="none") -> int:
    """One single-pattern pass (explorer.py:292-308)."""
    rules = [r for r in single_rules if not r.multi]
    filt, rep = saturate(eg, rules, ExploreLimits(n_max=1 << 62, k_max=1, k_multi=0), filter_mode,
                         filt=set() if filt is None else filt)
    return rep.total("applied")
