"""CPU-only checks of the C-ABI library and host logic (no device calls)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "tsat.h")).read()
    return sorted(set(re.findall(r"\b(tsat_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2101_01332_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libtsat.so not built")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing
    assert set(_declared()) == set(_lib.EXPORTED)


def test_rule_compiler_blob_shape():
    from paper_2101_01332_b200.rules import default_rules

    class FakeEG:
        def __init__(self):
            self.atoms = {}

        def _atom(self, a):
            return self.atoms.setdefault((type(a) is int, a), len(self.atoms))

        def _flush_atoms(self):
            pass

    from paper_2101_01332_b200.egraph import compile_ruleset

    blob, pidx = compile_ruleset(FakeEG(), list(default_rules()))
    assert len(pidx) == 13  # 18 sources -> 13 canonical patterns (reference test_rules.py:267-274)
    assert blob[0] == 13
