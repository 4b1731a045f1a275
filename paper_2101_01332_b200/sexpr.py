"""Terms and patterns (host side; input to the rule compiler).

Mirrors the reference term model (reference: pkg/src/tensorsat/sexpr.py:22-137):
``App(op, args)`` with ``op`` an int or str atom, ``Var(name)`` written ``?name``.
Integer-looking tokens become ``int`` atoms, everything else ``str``.
"""

from __future__ import annotations

import re
from dataclasses import dataclass
from typing import Iterator, Union

from .errors import SExprError

Atom = Union[int, str]


@dataclass(frozen=True)
class Var:
    name: str

    def __str__(self) -> str:
        return "?" + self.name


@dataclass(frozen=True)
class App:
    op: Atom
    args: tuple = ()

    def __str__(self) -> str:
        return format_term(self)


Term = Union[Var, App]

_LEX = re.compile(r"[()]|[^\s()]+")
_INTLIKE = re.compile(r"-?\d+\Z")


def _leaf(tok: str) -> Term:
    if tok[0] == "?":
        if len(tok) == 1:
            raise SExprError("empty variable name '?'")
        return Var(tok[1:])
    return App(int(tok)) if _INTLIKE.match(tok) else App(tok)


def parse_many(text: str) -> list[Term]:
    """All top-level expressions in ``text`` (reference: sexpr.py:66-102)."""
    toks = _LEX.findall(text)
    out: list[Term] = []
    # explicit stack of (head, args) frames instead of recursion
    i = 0
    n = len(toks)
    while i < n:
        tok = toks[i]
        i += 1
        if tok == ")":
            raise SExprError(f"unexpected ')' in {text!r}")
        if tok != "(":
            out.append(_leaf(tok))
            continue
        frames: list[tuple[Atom, list]] = []
        # open the first frame
        while True:
            if i >= n:
                raise SExprError(f"unclosed '(' in {text!r}")
            head = toks[i]
            i += 1
            if head in ("(", ")"):
                raise SExprError(f"operator expected after '(' in {text!r}")
            h = _leaf(head)
            if isinstance(h, Var):
                raise SExprError(f"variable {h} cannot be an operator")
            frames.append((h.op, []))
            # consume arguments until a nested '(' or the closing ')'
            done = None
            while frames:
                if i >= n:
                    raise SExprError(f"unclosed '(' in {text!r}")
                tok = toks[i]
                i += 1
                if tok == "(":
                    break  # nested frame: read its head in the outer loop
                if tok == ")":
                    op, args = frames.pop()
                    term = App(op, tuple(args))
                    if frames:
                        frames[-1][1].append(term)
                    else:
                        done = term
                        break
                else:
                    frames[-1][1].append(_leaf(tok))
            if done is not None:
                out.append(done)
                break
    return out


def parse(text: str) -> Term:
    terms = parse_many(text)
    if len(terms) != 1:
        raise SExprError(f"expected one expression, found {len(terms)}: {text!r}")
    return terms[0]


def format_term(t: Term) -> str:
    if isinstance(t, Var):
        return "?" + t.name
    if not t.args:
        return str(t.op)
    return "(" + " ".join([str(t.op), *(format_term(a) for a in t.args)]) + ")"


def walk(t: Term) -> Iterator[Term]:
    stack = [t]
    while stack:
        cur = stack.pop()
        yield cur
        if isinstance(cur, App):
            stack.extend(reversed(cur.args))


def variables(t: Term) -> list[str]:
    """Distinct variable names in first-occurrence pre-order."""
    seen: dict[str, None] = {}
    for sub in walk(t):
        if isinstance(sub, Var) and sub.name not in seen:
            seen[sub.name] = None
    return list(seen)


def is_ground(t: Term) -> bool:
    return not any(isinstance(s, Var) for s in walk(t))


def depth(t: Term) -> int:
    if isinstance(t, Var) or not t.args:
        return 1
    return 1 + max(depth(a) for a in t.args)
