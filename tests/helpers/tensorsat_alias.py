"""pytest plugin: makes ``import tensorsat.X`` resolve to this package, so the
reference's own test suite (copied to oracle/_ref/ref_tests by
__graft_entry__.build_reference) runs against the B200 engine unchanged.
Test infrastructure only (tests/test_reference_suite.py)."""

import importlib
import sys

import paper_2101_01332_b200 as _pkg

_MODULES = ["sexpr", "errors", "egraph", "tensor_lang", "rules", "cycles", "explorer", "cost", "extract", "cli"]

sys.modules["tensorsat"] = _pkg
for _m in _MODULES:
    sys.modules[f"tensorsat.{_m}"] = importlib.import_module(f"paper_2101_01332_b200.{_m}")
sys.modules["tensorsat.bench"] = importlib.import_module("paper_2101_01332_b200.bench_graphs")
_pkg.bench = sys.modules["tensorsat.bench"]
