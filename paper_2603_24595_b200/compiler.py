"""Site compiler: one checker query -> GPU search problems.

A site query is the assertion list the reference's checker hands its solver
(``engine/detectors.py:111-116`` overflow, ``:143-147`` bounds,
``:213-219`` race, ``:284`` deref).  The reference decides it with an exact
ILP procedure and then pins every symbol by bisection to the canonical
lexicographic optimum (``engine/report.py:147-203``).  This module turns the
query into data-parallel search problems whose lexicographic optimum over
a finite box *is* that canonical witness, and which the sm_100a engine
decides by interval branch-and-prune plus exhaustive leaf enumeration.

Steps (each exact: the model set and the witness order are preserved):

1. simplify and split into symbol-connected components exactly as the
   reference does (``solver/builtin.py:727-737``, ``:767-793``) so that the
   three-valued combination rule (unsat > unknown > sat,
   ``solver/builtin.py:737-750``) can be mirrored;
2. per component, mirror what the reference cannot decide: paths through a
   float atom or a non-constant shift are unsupported
   (``solver/linear.py:389-391``, ``:459-477``), a non-constant ``shr`` or a
   division by constant zero makes the whole component unsupported
   (``solver/linear.py:148-150``, ``:219-229``, ``:284-286``).  Unsupported
   atoms are replaced by FALSE in negation normal form; an empty remainder
   with such atoms present is ``unknown``;
3. presolve: linear normalisation, bound extraction, fixed-symbol folding,
   elimination of a symbol defined by a unit-coefficient equality (only when
   every other symbol of the equality precedes it in witness order, so the
   optimum over the remaining free symbols is unchanged), lattice
   substitution for ``emod(.., c) == r`` loop-summary atoms
   (``engine/executor.py:680-684``), gcd aggregation of wide equality terms,
   and interval bound tightening;
4. split the remaining atoms into independent problems and emit register
   bytecode for the device.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Set, Tuple

from . import ir, refmirror
from .ir import Node
from .order import optimization_order

INF = None  # unbounded side of an interval

# opcodes shared with csrc/mk_engine.cuh
OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MOD, OP_EMOD, OP_SHL, OP_SHR = 1, 2, 3, 4, 5, 6, 7, 8
OP_EQ, OP_NE, OP_LT, OP_LE, OP_GT, OP_GE = 16, 17, 18, 19, 20, 21
OP_AND, OP_OR, OP_NOT, OP_ITE = 32, 33, 34, 35
OP_ATOM = 40
_ARITH_OP = {"add": OP_ADD, "sub": OP_SUB, "mul": OP_MUL, "div": OP_DIV,
             "mod": OP_MOD, "emod": OP_EMOD, "shl": OP_SHL, "shr": OP_SHR}
_CMP_OP = {"eq": OP_EQ, "ne": OP_NE, "lt": OP_LT, "le": OP_LE, "gt": OP_GT, "ge": OP_GE}

MAX_VARS = 64        # free symbols per device problem (bit mask width)
# host-side FBBT over the presolved rows; off: bound propagation is left to
# the device's root contraction (mk_contract), measurement switch
HOST_FBBT = os.environ.get("MK_HOST_FBBT", "1") != "0"
# disjunctive contraction row groups (include/mk_b200.h mk_row.group), switch
ROW_GROUPS = os.environ.get("MK_ROW_GROUPS", "1") != "0"
# case split of a disjunction left after presolve (_split_disjunction), switch
OR_SPLIT = os.environ.get("MK_OR_SPLIT", "1") != "0"
MAX_REGS = 1024
MAX_TEMPS = 64       # temporaries of a search problem (mk_core.cuh MK_MAXT: flag bit masks)
_AGG_WIDE = 4096
_NEG = {"eq": "ne", "ne": "eq", "lt": "ge", "le": "gt", "gt": "le", "ge": "lt"}
_FLIP = {"lt": "gt", "le": "ge", "gt": "lt", "ge": "le", "eq": "eq", "ne": "ne"}


class CompileError(Exception):
    """The query is outside what the compiler handles; the site is reported
    ``unknown`` (mirrors the reference's honest-unknown convention)."""


class CapacityError(RuntimeError):
    """The query is decidable but exceeds a limit of this engine (free
    symbols per problem, registers, an unbounded symbol after presolve).
    The reference would decide it, so reporting ``unknown`` would break
    parity silently: this is an operational error and propagates to the
    caller (engine/detectors.py convention: operational errors surface as
    Python exceptions), never a verdict and never a fallback."""


# -- device problem --------------------------------------------------------------------

@dataclass
class Problem:
    """One independent lexicographic search over a box of free symbols."""

    var_names: List[str]           # free symbols in witness (position) order
    lo: List[int]
    hi: List[int]
    maximize: List[bool]
    insns: List[Tuple[int, int, int, int, int]] = field(default_factory=list)
    consts: List[int] = field(default_factory=list)
    nregs: int = 0
    atom_regs: List[int] = field(default_factory=list)
    atom_masks: List[int] = field(default_factory=list)
    # (rel, c0, [(var, coef)], group): include/mk_b200.h mk_row
    rows: List[Tuple[int, int, List[Tuple[int, int]], int]] = field(default_factory=list)
    ops_per_point: int = 0         # instructions evaluated per instance
    narrow: bool = False           # exact in 64-bit arithmetic (narrow_proof)
    any_model: bool = False        # feasibility only: stop at the first model

    @property
    def nvars(self) -> int:
        return len(self.var_names)

    def volume(self) -> int:
        v = 1
        for a, b in zip(self.lo, self.hi):
            v *= (b - a + 1)
        return v


@dataclass
class Group:
    """A raw (reference-level) component and the problems it compiled to."""

    status: str                    # "pending" | "unsat" | "unknown"
    reason: Optional[str]
    had_unsupported: bool
    problems: List[int] = field(default_factory=list)
    # disjunct branches (_split_disjunction): (problem indices, eliminated
    # symbol definitions, the component's symbols); the group's models are
    # the union of the branches' models
    alts: List[Tuple[List[int], Dict[str, Node], List[str]]] = field(default_factory=list)


@dataclass
class CompiledQuery:
    witness_names: List[str]
    order: List[Tuple[str, str]]
    groups: List[Group]
    problems: List[Problem]
    defs: Dict[str, Node]          # eliminated symbols -> expr over free symbols
    free_default: Dict[str, int]   # symbols absent from every atom
    compile_s: float = 0.0         # host time spent compiling this query

    @staticmethod
    def _status_of(idxs: Sequence[int], results) -> str:
        gs = "sat"
        for pi in idxs:
            st = results[pi][0]
            if st == "unsat":
                return "unsat"
            if st != "sat":
                gs = "unknown"
        return gs

    def _better(self, a: Dict[str, int], b: Dict[str, int], names: Sequence[str]) -> bool:
        """a precedes b in the canonical witness order (engine/report.py:
        177-203: ids max, everything else min) over the component's names."""
        inside = set(names)
        for n, d in self.order:
            if n not in inside or n not in a or n not in b or a[n] == b[n]:
                continue
            return a[n] > b[n] if d == "max" else a[n] < b[n]
        return False

    def assemble(self, results: Sequence[Tuple[str, Optional[List[int]]]]):
        """Combine per-problem device results into the reference verdict.

        Returns (status, witness) with status in sat/unsat/unknown."""
        status = "sat"
        pending_unknown = False
        for g in self.groups:
            if g.status == "unsat":
                return "unsat", {}
            if g.status == "unknown":
                pending_unknown = True
                continue
            if g.alts:
                sts = [self._status_of(idx, results) for idx, _, _ in g.alts]
                gs = ("unsat" if all(x == "unsat" for x in sts) else
                      "unknown" if any(x == "unknown" for x in sts) else "sat")
            else:
                gs = self._status_of(g.problems, results)
            if gs == "unsat":
                if g.had_unsupported:
                    pending_unknown = True
                    continue
                return "unsat", {}
            if gs == "unknown":
                pending_unknown = True
        if pending_unknown:
            return "unknown", {}
        binding: Dict[str, int] = dict(self.free_default)
        alt_members = {pi for g in self.groups for idx, _, _ in g.alts for pi in idx}
        for i, (p, (st, point)) in enumerate(zip(self.problems, results)):
            if i in alt_members:
                continue
            for name, v in zip(p.var_names, point):
                binding[name] = v
        for name, e in self.defs.items():
            binding[name] = ir.evaluate(e, binding)
        for g in self.groups:
            best = None
            for idx, defs, names in g.alts:
                if self._status_of(idx, results) != "sat":
                    continue
                b: Dict[str, int] = dict(self.free_default)
                for pi in idx:
                    for name, v in zip(self.problems[pi].var_names, results[pi][1]):
                        b[name] = v
                for name, e in defs.items():
                    b[name] = ir.evaluate(e, b)
                if best is None or self._better(b, best[0], names):
                    best = (b, names)
            if best is not None:
                for n in best[1]:
                    if n in best[0]:
                        binding[n] = best[0][n]
        witness = {n: binding[n] for n in sorted(self.witness_names) if n in binding}
        return status, witness


# -- linear forms ------------------------------------------------------------------------

LinForm = Tuple[Dict[object, int], int]   # term -> coeff, const ; term is str | opaque Node


def _lin_add(a: LinForm, b: LinForm, sign: int = 1) -> LinForm:
    out = dict(a[0])
    for k, c in b[0].items():
        v = out.get(k, 0) + sign * c
        if v:
            out[k] = v
        else:
            out.pop(k, None)
    return out, a[1] + sign * b[1]


def _proportional(a: LinForm, b: LinForm) -> Optional[int]:
    """k when a == k * b exactly (integer k, b non-constant), else None."""
    terms_b, c_b = b
    if not terms_b or set(a[0]) != set(terms_b):
        return None
    k = None
    for t, cb in terms_b.items():
        ca = a[0][t]
        if ca % cb:
            return None
        q = ca // cb
        if k is None:
            k = q
        elif q != k:
            return None
    if a[1] != k * c_b:
        return None
    return k


def _lin_scale(a: LinForm, f: int) -> LinForm:
    if f == 0:
        return {}, 0
    return {k: c * f for k, c in a[0].items()}, a[1] * f


def _term_sort_key(k) -> Tuple[int, str]:
    return (0, k) if isinstance(k, str) else (1, ir.render(k))


def lin_to_ir(lf: LinForm, widths: Dict[str, str]) -> Node:
    terms, c = lf
    acc: Optional[Node] = None
    for k in sorted(terms, key=_term_sort_key):
        coef = terms[k]
        t = ("s", k, widths.get(k, "i64")) if isinstance(k, str) else k
        if coef != 1:
            t = ("b", "mul", ("c", coef, "i64"), t, "i64")
        acc = t if acc is None else ("b", "add", acc, t, "i64")
    if acc is None:
        return ("c", c, "i64")
    if c:
        acc = ("b", "add", acc, ("c", c, "i64"), "i64")
    return acc


class _Lin:
    """Memoised linearisation of integer IR into linear forms over symbols
    and opaque nonlinear subterms (math-mode exact)."""

    def __init__(self, widths: Dict[str, str]) -> None:
        self.widths = widths
        self.memo: Dict[Node, LinForm] = {}

    def norm(self, e: Node) -> Node:
        return lin_to_ir(self.lin(e), self.widths)

    def lin(self, e: Node) -> LinForm:
        got = self.memo.get(e)
        if got is not None:
            return got
        r = self._lin(e)
        self.memo[e] = r
        return r

    def _opaque(self, e: Node) -> LinForm:
        return {e: 1}, 0

    def _lin(self, e: Node) -> LinForm:
        t = e[0]
        if t == "c":
            if not isinstance(e[1], int):
                raise CompileError("float constant in arithmetic")
            return {}, int(e[1])
        if t == "s":
            return {e[1]: 1}, 0
        if t == "x":
            return self.lin(e[1])
        if t == "b":
            op = e[1]
            la = self.lin(e[2])
            if op in ("add", "sub"):
                return _lin_add(la, self.lin(e[3]), 1 if op == "add" else -1)
            lb = self.lin(e[3])
            if op == "mul":
                if not la[0]:
                    return _lin_scale(lb, la[1])
                if not lb[0]:
                    return _lin_scale(la, lb[1])
                a = lin_to_ir(la, self.widths)
                b = lin_to_ir(lb, self.widths)
                if ir.render(a) > ir.render(b):
                    a, b = b, a
                return self._opaque(("b", "mul", a, b, "i64"))
            if op == "shl" and not lb[0] and 0 <= lb[1] <= 256:
                return _lin_scale(la, 1 << lb[1])
            if not lb[0] and not la[0]:
                try:
                    return {}, ir.apply_binop(op, la[1], lb[1])
                except ir.EvalError:
                    pass
            if op in ("div", "mod", "emod") and lb[0]:
                # k*B / B = k, k*B mod B = 0: exact wherever B != 0, and every
                # symbolic divisor of a component carries the side atom
                # B != 0 (compile_query; solver/linear.py:184-259), so no
                # model is gained or lost
                k = _proportional(la, lb)
                if k is not None:
                    return ({}, k) if op == "div" else ({}, 0)
            if op in ("div", "mod", "emod") and not lb[0] and lb[1] != 0:
                c = lb[1]
                if op == "emod":
                    m = abs(c)
                    terms = {}
                    for k, v in la[0].items():
                        r = v % m
                        if r > m // 2:
                            r -= m
                        if r:
                            terms[k] = r
                    if not terms:
                        return {}, la[1] % m
                    k0 = la[1] % m
                    inner = lin_to_ir((terms, k0), self.widths)
                    return self._opaque(("b", "emod", inner, ("c", m, "i64"), "i64"))
                if all(v % c == 0 for v in la[0].values()) and la[1] % c == 0:
                    if op == "div":
                        return {k: v // c for k, v in la[0].items()}, la[1] // c
                    return {}, 0
                inner = lin_to_ir(la, self.widths)
                return self._opaque(("b", op, inner, ("c", c, "i64"), "i64"))
            a = lin_to_ir(la, self.widths)
            b = lin_to_ir(lb, self.widths)
            return self._opaque(("b", op, a, b, "i64"))
        if t == "i":
            return self._opaque(e)
        raise CompileError(f"boolean node in arithmetic position: {e[0]}")


# -- interval helper (math mode, None = unbounded) ---------------------------------------------

def _imul(x, y):
    c = []
    for a in x:
        for b in y:
            if a is None or b is None:
                return (None, None)
            c.append(a * b)
    return (min(c), max(c))


def _tdiv(a, b):
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


class _Ivl:
    def __init__(self, bounds: Dict[str, Tuple[Optional[int], Optional[int]]]):
        self.bounds = bounds
        self.memo: Dict[Node, Tuple[Optional[int], Optional[int]]] = {}

    def __call__(self, e: Node):
        got = self.memo.get(e)
        if got is not None:
            return got
        r = self._go(e)
        self.memo[e] = r
        return r

    def _go(self, e: Node):
        t = e[0]
        if t == "c":
            return (e[1], e[1])
        if t == "s":
            return self.bounds.get(e[1], (None, None))
        if t == "x":
            return self(e[1])
        if t in ("p", "o"):
            return (0, 1)
        if t == "i":
            a, b = self(e[2]), self(e[3])
            lo = None if a[0] is None or b[0] is None else min(a[0], b[0])
            hi = None if a[1] is None or b[1] is None else max(a[1], b[1])
            return (lo, hi)
        op = e[1]
        x, y = self(e[2]), self(e[3])
        add = lambda p, q: None if p is None or q is None else p + q  # noqa: E731
        if op == "add":
            return (add(x[0], y[0]), add(x[1], y[1]))
        if op == "sub":
            return (add(x[0], None if y[1] is None else -y[1]),
                    add(x[1], None if y[0] is None else -y[0]))
        if op == "mul":
            return _imul(x, y)
        if op == "shl" and y[0] is not None and y[0] == y[1] and 0 <= y[0] <= 256:
            return _imul(x, (1 << y[0], 1 << y[0]))
        if op == "shr" and y[0] is not None and y[0] == y[1] and 0 <= y[0] <= 256:
            return (None if x[0] is None else x[0] >> y[0],
                    None if x[1] is None else x[1] >> y[0])
        if op == "emod" and y[0] is not None and y[0] == y[1] and y[0] != 0:
            return (0, abs(y[0]) - 1)
        if op == "div" and y[0] is not None and y[1] is not None and (y[0] >= 1 or y[1] <= -1):
            if x[0] is None or x[1] is None:
                return (None, None)
            c = [_tdiv(a, b) for a in x for b in y]
            return (min(c), max(c))
        if op == "mod" and y[0] is not None and y[0] == y[1] and y[0] != 0:
            m = abs(y[0]) - 1
            return (0 if (x[0] is not None and x[0] >= 0) else -m,
                    0 if (x[1] is not None and x[1] <= 0) else m)
        return (None, None)


# -- boolean normal form ------------------------------------------------------------------

def _has_float(e: Node) -> bool:
    t = e[0]
    if t in ("c", "s"):
        return ir.is_float(e[2])
    if t in ("b", "x", "i") and ir.is_float(ir.width_of(e)):
        return True
    if t == "x" and ir.is_float(ir.width_of(e[1])):
        return True
    return any(_has_float(c) for c in ir.children(e))


def _bad_shl(e: Node) -> bool:
    if e[0] == "b" and e[1] == "shl":
        r = e[3]
        if r[0] != "c" or not (0 <= r[1] <= 256):
            return True
    return any(_bad_shl(c) for c in ir.children(e))


def _component_unsupported(e: Node) -> Optional[str]:
    """Whole-component failures raised by the reference's ``rewrite_divs``
    (solver/linear.py:130-306)."""
    if e[0] == "b":
        op, r = e[1], e[3]
        if op == "shr" and (r[0] != "c" or not (0 <= r[1] <= 256)):
            return "unsupported: shift amount must be a small constant"
        if op in ("div", "mod") and r[0] == "c" and r[1] == 0:
            return "unsupported: division by constant zero"
        if op == "emod" and r[0] == "c" and r[1] == 0:
            return "unsupported: emod by constant zero"
    for c in ir.children(e):
        got = _component_unsupported(c)
        if got:
            return got
    return None


def _nnf(e: Node, neg: bool, flags: Dict[str, bool]) -> Node:
    """Negation normal form with unsupported atoms replaced by FALSE
    (the reference drops such paths, solver/builtin.py:815-821)."""
    t = e[0]
    if t == "c":
        v = 1 if e[1] else 0
        return ir.TRUE if (v ^ neg) else ir.FALSE
    if t == "o":
        if e[1] == "not":
            return _nnf(e[2][0], not neg, flags)
        op = e[1]
        if neg:
            op = "or" if op == "and" else "and"
        return ("o", op, tuple(_nnf(a, neg, flags) for a in e[2]))
    if t == "p":
        if _has_float(e) or _bad_shl(e):
            flags["unsupported"] = True
            return ir.FALSE
        op = _NEG[e[1]] if neg else e[1]
        return ("p", op, e[2], e[3])
    if t == "i":
        c_pos = _nnf(e[1], False, flags)
        c_neg = _nnf(e[1], True, flags)
        th = _nnf(e[2], neg, flags)
        ot = _nnf(e[3], neg, flags)
        return ("o", "or", (("o", "and", (c_pos, th)), ("o", "and", (c_neg, ot))))
    if t == "s" and e[2] == "bool":
        return ("p", "eq" if not neg else "ne", e, ("c", 1, "bool"))
    raise CompileError(f"cannot assert a {t} node")


def _symbolic_divisors(nodes) -> List[Node]:
    out: List[Node] = []
    seen: Set[Node] = set()
    stack = list(nodes)
    while stack:
        e = stack.pop()
        if e[0] == "b" and e[1] in ("div", "mod", "emod") and e[3][0] != "c":
            if e[3] not in seen:
                seen.add(e[3])
                out.append(e[3])
        stack.extend(ir.children(e))
    return out


def _may_err(e: Node) -> bool:
    """True when evaluating ``e`` can raise (symbolic or zero divisor)."""
    if e[0] == "b" and e[1] in ("div", "mod", "emod"):
        r = e[3]
        if not (r[0] == "c" and r[1] != 0):
            return True
    return any(_may_err(c) for c in ir.children(e))


def _truth(e: Node, ivl: "_Ivl") -> str:
    """Three-valued truth of a normalised boolean node over symbol bounds."""
    t = e[0]
    if t == "c":
        return "T" if e[1] else "F"
    if t == "p":
        a, b = ivl(e[2]), ivl(e[3])
        if None in a or None in b:
            lo = None if a[0] is None or b[1] is None else a[0] - b[1]
            hi = None if a[1] is None or b[0] is None else a[1] - b[0]
        else:
            lo, hi = a[0] - b[1], a[1] - b[0]
        op = e[1]
        if op == "le":
            if hi is not None and hi <= 0:
                return "T"
            if lo is not None and lo > 0:
                return "F"
        elif op == "lt":
            if hi is not None and hi < 0:
                return "T"
            if lo is not None and lo >= 0:
                return "F"
        elif op == "ge":
            if lo is not None and lo >= 0:
                return "T"
            if hi is not None and hi < 0:
                return "F"
        elif op == "gt":
            if lo is not None and lo > 0:
                return "T"
            if hi is not None and hi <= 0:
                return "F"
        elif op in ("eq", "ne"):
            tv = "?"
            if lo is not None and hi is not None and lo == hi == 0:
                tv = "T"
            elif (lo is not None and lo > 0) or (hi is not None and hi < 0):
                tv = "F"
            if op == "ne" and tv != "?":
                tv = "F" if tv == "T" else "T"
            return tv
        return "?"
    if t == "o":
        if e[1] == "not":
            v = _truth(e[2][0], ivl)
            return {"T": "F", "F": "T"}.get(v, "?")
        vals = [_truth(a, ivl) for a in e[2]]
        if e[1] == "and":
            if "F" in vals:
                return "F"
            return "T" if all(v == "T" for v in vals) else "?"
        if "T" in vals:
            return "T"
        return "F" if all(v == "F" for v in vals) else "?"
    return "?"


def linear_truth(a: Node, ivl: "_Ivl") -> str:
    """Truth of a comparison atom over a box with the comparison's two sides
    cancelled as one exact linear form (``(1024*k + t) - t`` is ``1024*k``):
    symbols contribute exact ranges, opaque nonlinear terms interval ones.
    'T' / 'F' when decided on the whole box, '?' otherwise."""
    if a[0] != "p":
        return "?"
    try:
        terms, c0 = _lin_add(_Lin({}).lin(a[2]), _Lin({}).lin(a[3]), -1)
    except CompileError:
        return "?"
    lo = hi = c0
    for k, c in terms.items():
        r = ivl.bounds.get(k, (None, None)) if isinstance(k, str) else ivl(k)
        if r[0] is None or r[1] is None:
            return "?"
        x, y = c * r[0], c * r[1]
        lo += min(x, y)
        hi += max(x, y)
    op = a[1]
    if op == "le":
        return "T" if hi <= 0 else ("F" if lo > 0 else "?")
    if op == "lt":
        return "T" if hi < 0 else ("F" if lo >= 0 else "?")
    if op == "ge":
        return "T" if lo >= 0 else ("F" if hi < 0 else "?")
    if op == "gt":
        return "T" if lo > 0 else ("F" if hi <= 0 else "?")
    if op == "eq":
        return "T" if lo == hi == 0 else ("F" if lo > 0 or hi < 0 else "?")
    if op == "ne":
        return "T" if lo > 0 or hi < 0 else ("F" if lo == hi == 0 else "?")
    return "?"


def _form_key(terms: Dict[object, int]) -> Tuple[Tuple, int]:
    """(normalised form, factor) with terms == factor * form, the form
    gcd-reduced with its first coefficient positive."""
    g = 0
    for v in terms.values():
        g = math.gcd(g, abs(v))
    first = min(terms, key=_term_sort_key)
    f = g if terms[first] > 0 else -g
    key = tuple(sorted(((k if isinstance(k, str) else ir.render(k)), v // f)
                       for k, v in terms.items()))
    return key, f


_NO_QUOTIENT = bool(__import__("os").environ.get("MK_NO_QUOTIENT"))   # measurement switches
_NO_RADIX = bool(__import__("os").environ.get("MK_NO_RADIX"))


def _replace_node(e: Node, old: Node, new: Node) -> Node:
    """Every occurrence of the subtree ``old`` in ``e`` replaced by ``new``."""
    if e == old:
        return new
    kids = ir.children(e)
    if not kids:
        return e
    repl = tuple(_replace_node(c, old, new) for c in kids)
    return e if repl == kids else ir.rebuild(e, repl)


# -- presolve ----------------------------------------------------------------------------

class _Presolve:
    def __init__(self, atoms: List[Node], widths: Dict[str, str],
                 pos: Dict[str, float], maximize: Dict[str, bool], light: bool = False) -> None:
        # light: structural steps only (normalisation, unary bounds, folding,
        # elimination, lattices); every step that reasons with the symbols'
        # ranges (bound tightening, dead disjuncts, quotients, radix split,
        # aggregation, relaxation / opposite rows, Fourier-Motzkin) is left to
        # the device search -- the first tier of SiteChecker.check_queries
        self.light = light
        self.widths = widths
        self.pos = pos
        self.maximize = maximize
        self.bounds: Dict[str, Tuple[Optional[int], Optional[int]]] = {}
        for n, w in widths.items():
            self.bounds[n] = ir.bounds(w)
        self.defs: Dict[str, Node] = {}
        self.atoms: List[Node] = list(dict.fromkeys(atoms))
        self.unsat = False
        self.kcount = 0
        self.fm_rounds = 0
        self.fbbt_passes = 0
        self.agg_done: Set[Tuple] = set()
        self._canon_memo: Dict[Tuple, Node] = {}
        # comparison atoms normalised in an earlier pass, by object identity
        # (the atom list keeps its objects across passes; hashing the nested
        # tuples for every memo lookup dominated the pass)
        self._norm_by_id: Dict[int, Tuple[Node, Node]] = {}
        # atom -> (normalised form key, factor), constant (or None): _form_bounds
        self._form_memo: Dict[Node, Tuple] = {}
        self.cuts: Set[Node] = set()
        self._lin_memo = _Lin(self.widths)

    def fork(self, atoms: List[Node]) -> "_Presolve":
        """A presolve of the same component continuing from this state with
        ``atoms`` (the disjunct split, _compile_query)."""
        q = _Presolve.__new__(_Presolve)
        q.light = self.light
        q.widths = dict(self.widths)
        q.pos = dict(self.pos)
        q.maximize = dict(self.maximize)
        q.bounds = dict(self.bounds)
        q.defs = dict(self.defs)
        q.atoms = list(dict.fromkeys(atoms))
        q.unsat = False
        q.kcount = self.kcount
        q.fm_rounds = 0
        q.fbbt_passes = 0
        q.agg_done = set(self.agg_done)
        q._canon_memo = {}
        q._norm_by_id = {}
        q._form_memo = {}
        q.cuts = set()         # a fresh cut budget for the branch's own rows
        q._lin_memo = _Lin(q.widths)
        return q

    # symbols of an IR node (memo-free; atoms are small)
    @staticmethod
    def _vars(e: Node) -> Set[str]:
        return set(ir.symbols_of(e))

    def _canon_cmp(self, lin: _Lin, op: str, l: Node, r: Node) -> Node:
        """Normalise ``l op r`` to ``L op' 0`` with op' in le/eq/ne (pure in
        its arguments, so memoised across presolve passes)."""
        key = (op, l, r)
        got = self._canon_memo.get(key)
        if got is None:
            got = self._canon_cmp_raw(lin, op, l, r)
            self._canon_memo[key] = got
        return got

    def _canon_cmp_raw(self, lin: _Lin, op: str, l: Node, r: Node) -> Node:
        lf = _lin_add(lin.lin(l), lin.lin(r), -1)
        terms, c = lf
        if op in ("gt", "ge"):
            terms, c = {k: -v for k, v in terms.items()}, -c
            op = "lt" if op == "gt" else "le"
        if op == "lt":
            c += 1
            op = "le"
        if not terms:
            ok = {"le": c <= 0, "eq": c == 0, "ne": c != 0}[op]
            return ir.TRUE if ok else ir.FALSE
        g = 0
        for v in terms.values():
            g = math.gcd(g, abs(v))
        if op == "le":
            terms = {k: v // g for k, v in terms.items()}
            c = -((-c) // g)          # ceil(c / g)
        else:
            if c % g:
                return ir.FALSE if op == "eq" else ir.TRUE
            terms = {k: v // g for k, v in terms.items()}
            c //= g
            first = min(terms, key=_term_sort_key)
            if terms[first] < 0:
                terms, c = {k: -v for k, v in terms.items()}, -c
        return ("p", op, lin_to_ir((terms, c), self.widths), ("c", 0, "i64"))

    def _normalize(self, e: Node, lin: _Lin, ivl: Optional["_Ivl"] = None) -> Node:
        t = e[0]
        if t == "p":
            got = self._norm_by_id.get(id(e))
            if got is not None and got[0] is e:
                return got[1]
            n = self._canon_cmp(lin, e[1], e[2], e[3])
            self._norm_by_id[id(e)] = (e, n)
            return n
        if t == "o":
            args = tuple(self._normalize(a, lin, ivl) for a in e[2])
            if ivl is not None and e[1] in ("and", "or"):
                # drop operands decided by the symbol bounds; only operands that
                # cannot raise (no symbolic divisor) may go, since an error in
                # an operand makes the whole point a non-model
                drop = "F" if e[1] == "or" else "T"
                absorb = "T" if e[1] == "or" else "F"
                kept = []
                for a in args:
                    tv = _truth(a, ivl)
                    if tv == absorb and not _may_err(a):
                        kept = None
                        break
                    if tv == drop and not _may_err(a):
                        continue
                    kept.append(a)
                if kept is None:
                    return ir.TRUE if e[1] == "or" else ir.FALSE
                if not kept:
                    return ir.FALSE if e[1] == "or" else ir.TRUE
                args = tuple(kept)
            return ir.simplify(("o", e[1], args))
        return e

    def _split_and(self, atoms: List[Node]) -> List[Node]:
        out: List[Node] = []
        for a in atoms:
            if a[0] == "o" and a[1] == "and":
                out.extend(self._split_and(list(a[2])))
            else:
                out.append(a)
        return out

    def _set_bound(self, v: str, lo, hi) -> bool:
        olo, ohi = self.bounds.get(v, (None, None))
        nlo = olo if lo is None else (lo if olo is None else max(olo, lo))
        nhi = ohi if hi is None else (hi if ohi is None else min(ohi, hi))
        if (nlo, nhi) != (olo, ohi):
            self.bounds[v] = (nlo, nhi)
            if nlo is not None and nhi is not None and nlo > nhi:
                self.unsat = True
            return True
        return False

    def _substitute(self, name: str, e: Node) -> None:
        self._substitute_many({name: e})

    def _substitute_many(self, m: Dict[str, Node]) -> None:
        """Replace every symbol of ``m`` at once; the replacements must not
        mention each other's symbols (constants, say)."""
        memo: Dict[Node, Node] = {}
        # only nodes that mention a replaced symbol are rewritten (symbol
        # sets are memoised per node for the query, so unchanged atoms cost
        # one lookup per pass)
        def sub(e: Node) -> Node:
            syms = ir.symbols_of(e)
            if not any(n in syms for n in m):
                return e
            return ir.substitute(e, m, memo)

        self.atoms = [sub(a) for a in self.atoms]
        for k in list(self.defs):
            self.defs[k] = sub(self.defs[k])
        self.defs.update(m)

    def _eliminate(self, name: str, e: Node) -> None:
        lo, hi = self.bounds.pop(name, (None, None))
        if lo is not None:
            self.atoms.append(("p", "ge", e, ("c", lo, "i64")))
        if hi is not None:
            self.atoms.append(("p", "le", e, ("c", hi, "i64")))
        self._substitute(name, e)

    def _lin_of_atom(self, lin: _Lin, a: Node) -> Optional[LinForm]:
        if a[0] == "p" and a[3] == ("c", 0, "i64"):
            return lin.lin(a[2])
        return None

    def run(self, max_iter: int = 200) -> None:
        for _ in range(max_iter):
            if self.unsat:
                return
            if not self._pass():
                return

    def _pass(self) -> bool:
        # linear forms are pure in the node (widths only grow: new lattice
        # symbols), so one memo serves every pass of this presolve
        lin = self._lin_memo
        ivl0 = None if self.light else _Ivl(self.bounds)
        # 1. normalise, split conjunctions, drop truths
        new_atoms: List[Node] = []
        for a in self._split_and(self.atoms):
            n = self._normalize(a, lin, ivl0)
            if n == ir.TRUE:
                continue
            if n == ir.FALSE:
                self.unsat = True
                return False
            if n[0] == "o" and n[1] == "and":
                new_atoms.extend(self._split_and([n]))
            else:
                new_atoms.append(n)
        changed = new_atoms != self.atoms
        self.atoms = list(dict.fromkeys(new_atoms))
        # 2. unary bounds
        kept: List[Node] = []
        for a in self.atoms:
            lf = self._lin_of_atom(lin, a)
            if lf is not None and len(lf[0]) == 1:
                (k, c), = lf[0].items()
                if isinstance(k, str) and a[1] in ("le", "eq"):
                    const = lf[1]
                    if a[1] == "eq":
                        if (-const) % c:
                            self.unsat = True
                            return False
                        v = (-const) // c
                        self._set_bound(k, v, v)
                    elif c > 0:
                        self._set_bound(k, None, (-const) // c)
                    else:
                        self._set_bound(k, -(const // c), None)
                    changed = True
                    if self.unsat:
                        return False
                    continue
            kept.append(a)
        self.atoms = kept
        # 3. fold fixed symbols
        fixed = [(n, b[0]) for n, b in self.bounds.items()
                 if b[0] is not None and b[0] == b[1]]
        if fixed:
            for n, _ in fixed:
                del self.bounds[n]
            self._substitute_many({n: ("c", v, "i64") for n, v in fixed})
            return True
        if changed:
            return True
        # 3b. mixed-radix split with a symbolic radix (before elimination
        # rewrites the digit equality into bounds)
        if not self.light and self._try_radix(lin):
            return True
        # 4. unit-coefficient equality elimination (order preserving)
        if self._try_eliminate(lin):
            return True
        # 5. lattice substitution for emod(.., c) == r
        if self._try_lattice(lin):
            return True
        if self.light:
            return False
        # 5b. quotient variables for divisions by positive constants
        if self._try_quotient(lin):
            return True
        # 6. gcd aggregation of wide terms
        if self._try_aggregate(lin):
            return True
        if self._try_aggregate_ineq(lin):
            return True
        # 6b. linear relaxations of rows with bounded nonlinear terms (cuts)
        if self._try_relax(lin):
            return True
        # 6c. opposite rows over one linear form that exclude each other
        if self._try_parallel(lin):
            return True
        # 7. Fourier-Motzkin implied rows (sound cuts, never remove models)
        if self._try_fm(lin):
            return True
        # 8. interval bound tightening (capped: slow creep is left to the device)
        if not HOST_FBBT or self.fbbt_passes >= 24:
            return False
        self.fbbt_passes += 1
        return self._fbbt(lin)

    def _free_deps(self, k) -> Set[str]:
        return {k} if isinstance(k, str) else self._vars(k)

    def _try_eliminate(self, lin: _Lin) -> bool:
        best = None
        for a in self.atoms:
            if a[0] != "p" or a[1] != "eq":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None:
                continue
            terms, c = lf
            opaque_vars: Set[str] = set()
            for k in terms:
                if not isinstance(k, str):
                    opaque_vars |= self._vars(k)
            cands = [k for k, v in terms.items()
                     if isinstance(k, str) and abs(v) == 1 and k not in opaque_vars]
            if not cands:
                continue
            v = max(cands, key=lambda n: self.pos[n])
            others: Set[str] = set(opaque_vars)
            for k in terms:
                if isinstance(k, str) and k != v:
                    others.add(k)
            if any(self.pos[o] >= self.pos[v] for o in others):
                continue
            coef = terms[v]
            rest = {k: -x * coef for k, x in terms.items() if k != v}
            expr = lin_to_ir((rest, -c * coef), self.widths)
            if best is None or self.pos[v] > self.pos[best[0]]:
                best = (v, expr)
        if best is None:
            return False
        self._eliminate(best[0], best[1])
        return True

    def _try_lattice(self, lin: _Lin) -> bool:
        for idx, a in enumerate(self.atoms):
            if a[0] != "p" or a[1] != "eq":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None or len(lf[0]) != 1:
                continue
            (k, c1), = lf[0].items()
            if isinstance(k, str) or k[0] != "b" or k[1] != "emod" or abs(c1) != 1 \
                    or k[3][0] != "c":
                continue
            m = k[3][1]
            r = -lf[1] * c1
            if not 0 <= r < m:
                self.unsat = True
                return True
            inner = lin.lin(k[2])
            terms, k0 = inner
            opaque_vars: Set[str] = set()
            for t in terms:
                if not isinstance(t, str):
                    opaque_vars |= self._vars(t)
            cands = [t for t, v in terms.items()
                     if isinstance(t, str) and abs(v) == 1 and t not in opaque_vars]
            if not cands:
                continue
            v = max(cands, key=lambda n: self.pos[n])
            others = set(opaque_vars) | {t for t in terms if isinstance(t, str) and t != v}
            if any(self.pos[o] >= self.pos[v] for o in others):
                continue
            av = terms[v]
            # av*v + R + k0 = m*kk + r  ->  v = av*(m*kk + r - k0 - R)
            kname = f"{v}#k{self.kcount}"
            self.kcount += 1
            self.widths[kname] = "i64"
            self.pos[kname] = self.pos[v] - 0.25
            self.maximize[kname] = self.maximize.get(v, False) ^ (av < 0)
            # the lattice coordinate's range implied by v's range and the rest
            # of the index (kk = (av*v + k0 + R - r) / m): exact interval
            # arithmetic, so the light presolve (no tightening passes) still
            # hands the device a bounded box
            kb: Tuple[Optional[int], Optional[int]] = (None, None)
            vlo, vhi = self.bounds.get(v, (None, None))
            others_lf = ({t: x for t, x in terms.items() if t != v}, k0 - r)
            olo, ohi = _Ivl(self.bounds)(lin_to_ir(others_lf, self.widths)) \
                if others_lf[0] else (others_lf[1], others_lf[1])
            if None not in (vlo, vhi, olo, ohi):
                nlo = min(av * vlo, av * vhi) + olo
                nhi = max(av * vlo, av * vhi) + ohi
                kb = (-((-nlo) // m), nhi // m)
            self.bounds[kname] = kb
            rest = {t: -x * av for t, x in terms.items() if t != v}
            rest[kname] = m * av
            expr = lin_to_ir((rest, (r - k0) * av), self.widths)
            del self.atoms[idx]
            self._eliminate(v, expr)
            return True
        return False

    def _try_quotient(self, lin: _Lin) -> bool:
        """Quotient variable for a division by a positive constant whose
        dividend is linear and non-negative on the whole box (so truncation
        is the floor): q = e / d  <=>  d*q <= e <= d*q + d - 1, the rows the
        reference's own rewrite_divs introduces (solver/linear.py:130-306).
        Every occurrence of the quotient becomes q, so atoms that compared
        through it become linear rows the device's contraction (FBBT) can
        use.  q is a function of e's symbols; placed after every symbol in
        the witness order it changes neither the model set over the query's
        symbols nor its lexicographic optimum, and it is not a witness
        symbol.  Division by a positive constant cannot raise."""
        if self.kcount > 64 or _NO_QUOTIENT:
            return False
        ivl = _Ivl(self.bounds)
        seen: Set[Node] = set()
        for a in self.atoms:
            if a[0] != "p":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None:
                continue
            for k in lf[0]:
                if isinstance(k, str) or k in seen:
                    continue
                seen.add(k)
                if k[0] != "b" or k[1] != "div" or k[3][0] != "c" or not isinstance(k[3][1], int) \
                        or k[3][1] < 2:
                    continue
                d, e = k[3][1], k[2]
                ef = lin.lin(e)
                if not ef[0] or any(not isinstance(t, str) for t in ef[0]):
                    continue
                lo, hi = ivl(e)
                if lo is None or hi is None or lo < 0:
                    continue
                qname = f"{min(ef[0], key=_term_sort_key)}#q{self.kcount}"
                self.kcount += 1
                self.widths[qname] = "i64"
                self.pos[qname] = max(self.pos.values()) + 1.0
                self.maximize[qname] = False
                self.bounds[qname] = (lo // d, hi // d)
                q = ("s", qname, "i64")
                self.atoms = [_replace_node(x, k, q) for x in self.atoms]
                dq = ("b", "mul", ("c", d, "i64"), q, "i64")
                self.atoms.append(("p", "le", dq, e))
                self.atoms.append(("p", "le", e, ("b", "add", dq, ("c", d - 1, "i64"), "i64")))
                return True
        return False

    def _nonneg(self, x: str) -> bool:
        lo = self.bounds.get(x, (None, None))[0]
        return lo is not None and lo >= 0

    def _below(self, lin: _Lin, u: str, pname: str) -> bool:
        """Some atom states u <= P - k with k >= 1."""
        for a in self.atoms:
            if a[0] != "p" or a[1] != "le":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is not None and lf[0] == {u: 1, pname: -1} and lf[1] >= 1:
                return True
        return False

    def _try_radix(self, lin: _Lin) -> bool:
        """``c*P*X1 - c*P*X2 + R = 0`` with P a symbol >= 1 and R provably
        inside (-|c|*P, |c|*P): then P*(X1 - X2) is a multiple of P strictly
        inside (-P, P), so X1 = X2 and R = 0 (exact for integers).  R may hold
        one digit pair c_s*(u - w) with 0 <= u, w <= P - 1 (atoms), |c_s| <=
        |c|, plus terms of constant range K < |c_s| (or K < |c|*P_lo without
        a pair).  This is the injectivity of a mixed-radix index with a
        launch-dependent radix (``((seq * heads + head) * gridDim.z +
        blockIdx.z) * 128 + tid``), which a race twin query's offset
        equality hinges on; interval search cannot see it."""
        if _NO_RADIX:
            return False
        for idx, a in enumerate(self.atoms):
            if a[0] != "p" or a[1] != "eq":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None:
                continue
            terms, c0 = lf
            muls = [(k, v) for k, v in terms.items()
                    if not isinstance(k, str) and k[0] == "b" and k[1] == "mul"]
            if len(muls) != 2:
                continue
            (t1, c1), (t2, c2) = muls
            if c1 != -c2:
                continue
            common = [f for f in (t1[2], t1[3]) if f[0] == "s" and f in (t2[2], t2[3])]
            if len(common) != 1:
                continue
            P = common[0]
            pname = P[1]
            plo = self.bounds.get(pname, (None, None))[0]
            if plo is None or plo < 1:
                continue
            x1 = t1[2] if t1[3] == P else t1[3]
            x2 = t2[2] if t2[3] == P else t2[3]
            rest = {k: v for k, v in terms.items() if k not in (t1, t2)}
            # a bare P*X1 = P*X2 (no digit) is left to the search: splitting it
            # measured slower there (moe_align's twin offsets, 19 -> 26 ms)
            if not rest or any(not isinstance(k, str) for k in rest):
                continue
            # one digit pair below the radix
            pair = None
            for u, cu in rest.items():
                for w, cw in rest.items():
                    if u < w and cu == -cw and pair is None \
                            and all(self._nonneg(x) for x in (u, w)) \
                            and self._below(lin, u, pname) and self._below(lin, w, pname):
                        pair = (u, w, abs(cu))
            others = {k: v for k, v in rest.items() if pair is None or k not in pair[:2]}
            lo = hi = c0
            ok = True
            for k, v in others.items():
                b = self.bounds.get(k, (None, None))
                if b[0] is None or b[1] is None:
                    ok = False
                    break
                lo += min(v * b[0], v * b[1])
                hi += max(v * b[0], v * b[1])
            if not ok:
                continue
            K = max(abs(lo), abs(hi))
            if pair is not None:
                if not (pair[2] <= abs(c1) and K < pair[2]):
                    continue
            elif not K < abs(c1) * plo:
                continue
            del self.atoms[idx]
            self.atoms.append(("p", "eq", x1, x2))
            self.atoms.append(("p", "eq", lin_to_ir((rest, c0), self.widths), ("c", 0, "i64")))
            return True
        return False

    def _try_aggregate(self, lin: _Lin) -> bool:
        ivl = _Ivl(self.bounds)
        existing = set(self.atoms)
        for a in self.atoms:
            if a[0] != "p" or a[1] != "eq":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None:
                continue
            terms, c = lf
            wide, rlo, rhi = [], c, c
            for k, v in terms.items():
                if isinstance(k, str):
                    lo, hi = self.bounds.get(k, (None, None))
                else:
                    lo, hi = ivl(k)
                if isinstance(k, str) and (lo is None or hi is None or hi - lo > _AGG_WIDE):
                    wide.append(k)
                    continue
                if lo is None or hi is None:
                    rlo = rhi = None
                    break
                if rlo is not None:
                    rlo += min(v * lo, v * hi)
                    rhi += max(v * lo, v * hi)
            if rlo is None or not wide or len(wide) == len(terms):
                continue
            g = 0
            for k in wide:
                g = math.gcd(g, abs(terms[k]))
            if g <= 1:
                continue
            w_lo = -((rhi) // g)   # ceil(-rhi/g)
            w_hi = (-rlo) // g
            if w_lo > w_hi:
                self.unsat = True
                return True
            if w_lo != w_hi:
                continue
            wt = {k: terms[k] // g for k in wide}
            new = self._canon_cmp(lin, "eq", lin_to_ir((wt, -w_lo), self.widths), ("c", 0, "i64"))
            if new == ir.FALSE:
                self.unsat = True
                return True
            if new != ir.TRUE and new not in existing:
                self.atoms.append(new)
                return True
        return False

    def _form_bounds(self, lin: _Lin) -> Dict[Tuple, List]:
        """Bounds that single rows state on a normalised linear form
        (gcd-reduced, first coefficient positive)."""
        out: Dict[Tuple, List] = {}
        memo = self._form_memo
        for a in self.atoms:
            if a[0] != "p" or a[1] not in ("le", "eq"):
                continue
            got = memo.get(a)
            if got is None:
                lf = self._lin_of_atom(lin, a)
                got = memo[a] = (None,) if lf is None or not lf[0] else \
                    (_form_key(lf[0]), lf[1])
            if got[0] is None:
                continue
            (key, f), c = got
            ent = out.setdefault(key, [None, None])
            # f*F0 + c <= 0
            if f > 0:
                ub = (-c) // f
                ent[1] = ub if ent[1] is None else min(ent[1], ub)
            else:
                lb = -(c // f)
                ent[0] = lb if ent[0] is None else max(ent[0], lb)
            if a[1] == "eq":
                if f > 0:
                    lb = -(c // f)
                    ent[0] = lb if ent[0] is None else max(ent[0], lb)
                else:
                    ub = (-c) // f
                    ent[1] = ub if ent[1] is None else min(ent[1], ub)
        return out

    def _try_aggregate_ineq(self, lin: _Lin) -> bool:
        """Per wide linear form W (terms with range > 4096, common gcd g),
        intersect the W-bounds every row implies; a singleton becomes the
        equality W == w (the reference's row aggregation, applied to
        inequalities too), a tighter range becomes two implied rows.  The
        narrow remainder's range uses symbol bounds and any row bounding
        the same linear form."""
        ivl = _Ivl(self.bounds)
        fb = self._form_bounds(lin)
        acc: Dict[Tuple, List] = {}
        for a in self.atoms:
            if a[0] != "p" or a[1] not in ("le", "eq"):
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None:
                continue
            terms, c = lf
            wide, rlo, rhi = [], 0, 0
            narrow: Dict[object, int] = {}
            for k, v in terms.items():
                lo, hi = self.bounds.get(k, (None, None)) if isinstance(k, str) else ivl(k)
                if isinstance(k, str) and (lo is None or hi is None or hi - lo > _AGG_WIDE):
                    wide.append(k)
                    continue
                narrow[k] = v
                if lo is None or hi is None:
                    rlo = rhi = None
                    continue
                if rlo is not None:
                    rlo += min(v * lo, v * hi)
                    rhi += max(v * lo, v * hi)
            if narrow and len(narrow) > 1:
                key, f = _form_key(narrow)
                got = fb.get(key)
                if got is not None:
                    lo0, hi0 = got
                    cands = [x * f for x in (lo0, hi0) if x is not None]
                    if lo0 is not None and hi0 is not None:
                        nlo, nhi = min(cands), max(cands)
                    elif len(cands) == 1:
                        nlo, nhi = (cands[0], None) if (f > 0) == (lo0 is not None) else (None, cands[0])
                    else:
                        nlo = nhi = None
                    if rlo is None:
                        rlo, rhi = nlo, nhi
                    else:
                        if nlo is not None:
                            rlo = max(rlo, nlo)
                        if nhi is not None:
                            rhi = min(rhi, nhi)
            if rlo is None or rhi is None:
                continue
            rlo += c
            rhi += c
            if rlo is None or not wide or len(wide) == len(terms):
                continue
            g = 0
            for k in wide:
                g = math.gcd(g, abs(terms[k]))
            wt = {k: terms[k] // g for k in wide}
            first = min(wt, key=_term_sort_key)
            sign = 1 if wt[first] > 0 else -1
            key = tuple(sorted((k, sign * v) for k, v in wt.items()))
            # g*sign*W' + R <= 0  with W' = sign*wt
            ent = acc.setdefault(key, [None, None])
            ub = (-rlo) // g                      # g*w <= -R  =>  w <= floor(-rlo/g)
            if sign > 0:
                ent[1] = ub if ent[1] is None else min(ent[1], ub)
            else:
                lb = -ub
                ent[0] = lb if ent[0] is None else max(ent[0], lb)
            if a[1] == "eq":
                lb2 = -((rhi) // g)               # w >= ceil(-rhi/g)
                if sign > 0:
                    ent[0] = lb2 if ent[0] is None else max(ent[0], lb2)
                else:
                    ent[1] = -lb2 if ent[1] is None else min(ent[1], -lb2)
        existing = set(self.atoms)
        added = False
        for key, (lo, hi) in acc.items():
            if lo is not None and hi is not None and lo > hi:
                self.unsat = True
                return True
            wt = dict(key)
            if lo is not None and hi is not None and 0 < hi - lo <= _AGG_WIDE \
                    and key not in self.agg_done:
                # name the narrow combination: v := cv*(w - rest) for the last
                # unit-coefficient symbol v of W, w taking v's witness slot
                cands = [k for k, c in wt.items() if abs(c) == 1]
                if cands:
                    v = max(cands, key=lambda n: self.pos[n])
                    if all(self.pos[o] < self.pos[v] for o in wt if o != v):
                        self.agg_done.add(key)
                        cv = wt[v]
                        wname = f"{v}#w{self.kcount}"
                        self.kcount += 1
                        self.widths[wname] = "i64"
                        self.pos[wname] = self.pos[v] - 0.25
                        self.maximize[wname] = self.maximize.get(v, False) ^ (cv < 0)
                        self.bounds[wname] = (lo, hi)
                        rest = {k: -c * cv for k, c in wt.items() if k != v}
                        rest[wname] = cv
                        self._eliminate(v, lin_to_ir((rest, 0), self.widths))
                        return True
            wl = lin_to_ir((wt, 0), self.widths)
            cur = ivl(wl)
            news = []
            if lo is not None and hi is not None and lo == hi:
                news.append(self._canon_cmp(lin, "eq", wl, ("c", lo, "i64")))
            else:
                if hi is not None and (cur[1] is None or hi < cur[1]):
                    news.append(self._canon_cmp(lin, "le", wl, ("c", hi, "i64")))
                if lo is not None and (cur[0] is None or lo > cur[0]):
                    news.append(self._canon_cmp(lin, "ge", wl, ("c", lo, "i64")))
            for n in news:
                if n == ir.FALSE:
                    self.unsat = True
                    return True
                if n != ir.TRUE and n not in existing and n not in self.cuts:
                    self.cuts.add(n)
                    self.atoms.append(n)
                    existing.add(n)
                    added = True
        return added

    def _try_relax(self, lin: _Lin, max_new: int = 16) -> bool:
        """For a row whose nonlinear (opaque) terms are bounded on the
        current box, add the row with each such term replaced by the end of
        its range that weakens the row: implied by the row, so the model
        set is unchanged, and linear, so gcd aggregation, Fourier-Motzkin
        and bound propagation can use it (paged attention's partition-local
        logits index: 16*(4k + w - 32z) + (tx % 32) % 16 >= 512 relaxes to
        4k + w - 32z >= 32)."""
        ivl = _Ivl(self.bounds)
        existing = set(self.atoms)
        added = 0
        for a in list(self.atoms):
            if a[0] != "p" or a[1] != "le":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None:
                continue
            terms, c = lf
            opq = [(k, v) for k, v in terms.items() if not isinstance(k, str)]
            sym = {k: v for k, v in terms.items() if isinstance(k, str)}
            if not opq or not sym:
                continue
            shift = 0
            for k, v in opq:
                lo, hi = ivl(k)
                if lo is None or hi is None:
                    shift = None
                    break
                shift += min(v * lo, v * hi)
            if shift is None:
                continue
            n = self._canon_cmp(lin, "le", lin_to_ir((sym, c + shift), self.widths),
                                ("c", 0, "i64"))
            if n == ir.FALSE:
                self.unsat = True
                return True
            if n == ir.TRUE or n in existing or n in self.cuts:
                continue
            self.cuts.add(n)
            existing.add(n)
            self.atoms.append(n)
            added += 1
            if added >= max_new:
                break
        return added > 0

    def _try_parallel(self, lin: _Lin) -> bool:
        """f <= u and -f <= -l over the same symbols with l > u: no model
        (two rows of one linear form -- a relaxation cut against a
        Fourier-Motzkin row, say -- that bound propagation would only creep
        towards one unit per sweep).  Opaque terms (a product of symbols,
        say) count as one more coordinate: a term is a function of the
        symbols, so at any model both rows hold with the same value of it
        (a point where it raises is no model)."""
        upper: Dict[Tuple, int] = {}
        for a in self.atoms:
            if a[0] != "p" or a[1] != "le":
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None or not lf[0]:
                continue
            key = tuple(sorted(((k if isinstance(k, str) else ir.render(k)), v)
                               for k, v in lf[0].items()))
            u = -lf[1]                       # sum(terms) <= -c
            if key not in upper or u < upper[key]:
                upper[key] = u
        for key, u in upper.items():
            neg = tuple(sorted((k, -v) for k, v in key))
            if neg in upper and -upper[neg] > u:   # sum >= -u_neg > u
                self.unsat = True
                return True
        return False

    def _try_fm(self, lin: _Lin, max_terms: int = 3, max_new: int = 16) -> bool:
        """Add Fourier-Motzkin combinations of pairs of linear rows that
        cancel one symbol.  Non-negative combinations of rows are implied by
        them, so the model set is unchanged; the new rows let bound
        propagation and the device contraction see relational facts such as
        bx < SL and 4096*bx + idx >= 4096*SL  =>  idx >= 4096."""
        if self.fm_rounds >= 8:
            return False
        self.fm_rounds += 1
        rows: List[Tuple[Dict[str, int], int]] = []
        for a in self.atoms:
            if a[0] != "p" or a[1] not in ("le", "eq"):
                continue
            lf = self._lin_of_atom(lin, a)
            if lf is None:
                continue
            rows.append(lf)   # opaque product terms combine like symbols
            if a[1] == "eq":
                rows.append(({k: -v for k, v in lf[0].items()}, -lf[1]))
        existing = set(self.atoms)
        added = 0
        def wide(n: str) -> bool:
            lo, hi = self.bounds.get(n, (None, None))
            return lo is None or hi is None or hi - lo > _AGG_WIDE

        # only wide symbols are eliminated: narrow ones are cheap to enumerate
        symbols = sorted({k for t, _ in rows for k in t if isinstance(k, str) and wide(k)},
                         key=lambda n: self.pos.get(n, 0))
        # opaque terms (products of symbols, quotients) are eliminated too,
        # after the symbols: a term is one value at any model, so rows that
        # bound it from both sides imply their combination without it
        symbols += sorted({k for t, _ in rows for k in t if not isinstance(k, str)},
                          key=ir.render)
        if len(self.cuts) >= 48:
            return False
        for v in symbols:
            pos_rows = [r for r in rows if r[0].get(v, 0) > 0]
            neg_rows = [r for r in rows if r[0].get(v, 0) < 0]
            for p in pos_rows:
                for q in neg_rows:
                    a, b = p[0][v], -q[0][v]
                    comb = _lin_add(_lin_scale(p, b), _lin_scale(q, a))
                    if not comb[0]:
                        if comb[1] > 0:
                            self.unsat = True
                            return True
                        continue
                    if len(comb[0]) > max_terms:
                        continue
                    n = self._canon_cmp(lin, "le", lin_to_ir(comb, self.widths), ("c", 0, "i64"))
                    if n == ir.FALSE:
                        self.unsat = True
                        return True
                    if n == ir.TRUE or n in existing or n in self.cuts:
                        continue
                    self.cuts.add(n)
                    existing.add(n)
                    self.atoms.append(n)
                    added += 1
                    if added >= max_new:
                        return True
        return added > 0

    def _fbbt(self, lin: _Lin, rounds: int = 8) -> bool:
        any_change = False
        # the rows do not change inside the sweeps, only the bounds do
        rows = []
        for a in self.atoms:
            lf = self._lin_of_atom(lin, a)
            if lf is None or a[1] == "ne":
                continue
            rows.append((a, lf[0], lf[1]))
        for _ in range(rounds):
            ivl = _Ivl(self.bounds)
            changed = False
            for a, terms, c in rows:
                parts = []
                # activity range of the row: finite sums plus the number of
                # unbounded contributions, so each term's residual range is
                # the total less its own contribution (linear in the terms)
                smin = smax = c
                nmin = nmax = 0
                for k, v in terms.items():
                    lo, hi = self.bounds.get(k, (None, None)) if isinstance(k, str) else ivl(k)
                    mn, mx = (lo, hi) if v > 0 else (hi, lo)
                    mn = None if mn is None else v * mn
                    mx = None if mx is None else v * mx
                    if mn is None:
                        nmin += 1
                    else:
                        smin += mn
                    if mx is None:
                        nmax += 1
                    else:
                        smax += mx
                    parts.append((k, v, mn, mx))
                for k, v, mn, mx in parts:
                    if not isinstance(k, str):
                        continue
                    if mn is None:
                        rlo = smin if nmin == 1 else None
                    else:
                        rlo = smin - mn if nmin == 0 else None
                    if mx is None:
                        rhi = smax if nmax == 1 else None
                    else:
                        rhi = smax - mx if nmax == 0 else None
                    # v*x + rest <= 0  (and >= 0 for eq)
                    nlo = nhi = None
                    if rlo is not None:
                        if v > 0:
                            nhi = (-rlo) // v
                        else:
                            nlo = -(rlo // v)            # ceil(-rlo / v)
                    if a[1] == "eq" and rhi is not None:
                        if v > 0:
                            nlo = -(rhi // v)            # ceil(-rhi / v)
                        else:
                            nhi = (-rhi) // v            # floor(-rhi / v)
                    if self._set_bound(k, nlo, nhi):
                        changed = True
                        if self.unsat:
                            return True
            if not changed:
                break
            any_change = True
        return any_change


# -- bytecode emission -------------------------------------------------------------------

class _Emitter:
    def __init__(self, var_index: Dict[str, int]) -> None:
        self.var_index = var_index
        self.nvars = len(var_index)
        self.consts: List[int] = []
        self.const_reg: Dict[int, int] = {}
        self.code: List[List[int]] = []      # [op, dst, a, b, c] with virtual regs
        self.memo: Dict[Node, int] = {}
        self.next_v = 0

    def _const(self, v: int) -> int:
        r = self.const_reg.get(v)
        if r is None:
            r = -(len(self.consts) + 1)        # negative = const slot
            self.consts.append(v)
            self.const_reg[v] = r
        return r

    def _tmp(self) -> int:
        self.next_v += 1
        return 1_000_000 + self.next_v

    def emit(self, e: Node) -> int:
        got = self.memo.get(e)
        if got is not None:
            return got
        t = e[0]
        if t == "c":
            r = self._const(int(e[1]))
        elif t == "s":
            r = ("V", self.var_index[e[1]])
        elif t == "x":
            r = self.emit(e[1])
        elif t == "b":
            a = self.emit(e[2])
            b = self.emit(e[3])
            r = self._tmp()
            self.code.append([_ARITH_OP[e[1]], r, a, b, 0])
        elif t == "p":
            a = self.emit(e[2])
            b = self.emit(e[3])
            r = self._tmp()
            self.code.append([_CMP_OP[e[1]], r, a, b, 0])
        elif t == "o":
            if e[1] == "not":
                a = self.emit(e[2][0])
                r = self._tmp()
                self.code.append([OP_NOT, r, a, 0, 0])
            else:
                op = OP_AND if e[1] == "and" else OP_OR
                r = self.emit(e[2][0])
                for arg in e[2][1:]:
                    b = self.emit(arg)
                    d = self._tmp()
                    self.code.append([op, d, r, b, 0])
                    r = d
        elif t == "i":
            c = self.emit(e[1])
            a = self.emit(e[2])
            b = self.emit(e[3])
            r = self._tmp()
            self.code.append([OP_ITE, r, c, a, b])
        else:
            raise CompileError(f"cannot emit {t}")
        self.memo[e] = r
        return r

    def atom(self, e: Node, index: int) -> None:
        r = self.emit(e)
        self.code.append([OP_ATOM, 0, r, index, 0])

    def finish(self, atom_vregs: List[object]) -> Tuple[List[Tuple[int, int, int, int, int]], int, List[int]]:
        """Resolve virtual registers with a linear-scan allocator."""
        base = self.nvars + len(self.consts)

        def phys_fixed(r) -> Optional[int]:
            if isinstance(r, tuple):
                return r[1]
            if isinstance(r, int) and r < 0:
                return self.nvars + (-r - 1)
            return None

        # atoms must survive to the end
        last_use: Dict[int, int] = {}
        for i, ins in enumerate(self.code):
            opnds = ins[2:3] if ins[0] == OP_ATOM else ins[2:5]
            for opnd in opnds:
                if isinstance(opnd, int) and opnd >= 1_000_000:
                    last_use[opnd] = i
        end = len(self.code)
        for r in atom_vregs:
            if isinstance(r, int) and r >= 1_000_000:
                last_use[r] = end
        free: List[int] = []
        nphys = base
        assign: Dict[int, int] = {}
        out: List[Tuple[int, int, int, int, int]] = []
        for i, ins in enumerate(self.code):
            op, d, a, b, c = ins

            def res(x):
                f = phys_fixed(x)
                if f is not None:
                    return f
                if isinstance(x, int) and x >= 1_000_000:
                    return assign[x]
                return 0
            if op == OP_ATOM:
                pa = res(a)
                if isinstance(a, int) and a >= 1_000_000 and last_use.get(a) == i and a in assign:
                    free.append(assign.pop(a))
                out.append((op, 0, pa, b, 0))
                continue
            pa, pb = res(a), res(b) if op != OP_NOT else 0
            pc = res(c) if op == OP_ITE else 0
            # release operands whose last use is here
            for x in (a, b, c):
                if isinstance(x, int) and x >= 1_000_000 and last_use.get(x) == i and x in assign:
                    free.append(assign.pop(x))
            if free:
                pd = free.pop()
            else:
                pd = nphys
                nphys += 1
            assign[d] = pd
            if d not in last_use:   # dead value: release immediately
                free.append(assign.pop(d))
            out.append((op, pd, pa, pb, pc))
        atom_regs = []
        for r in atom_vregs:
            f = phys_fixed(r)
            atom_regs.append(f if f is not None else assign[r])
        if nphys > MAX_REGS:
            raise CapacityError(f"site needs {nphys} registers (> {MAX_REGS})")
        return out, nphys, atom_regs


def _le_forms(lin: "_Lin", e: Node):
    """A comparison as linear forms (rel, c0, terms) over symbols and opaque
    terms: sum <= 0 (rel 0) or sum == 0 (rel 1); ``ne`` is its two strict
    sides.  None when ``e`` is not a comparison of linear forms."""
    if e[0] != "p":
        return None
    try:
        terms, c0 = _lin_add(lin.lin(e[2]), lin.lin(e[3]), -1)
    except CompileError:
        return None
    if not terms:
        return None
    neg = {k: -v for k, v in terms.items()}
    op = e[1]
    if op == "le":
        return [(0, c0, terms)]
    if op == "lt":
        return [(0, c0 + 1, terms)]
    if op == "ge":
        return [(0, -c0, neg)]
    if op == "gt":
        return [(0, -c0 + 1, neg)]
    if op == "eq":
        return [(1, c0, terms)]
    if op == "ne":
        return [(0, c0 + 1, terms), (0, -c0 + 1, neg)]
    return None


def _relax(form, ivl: "_Ivl"):
    """Contraction rows implied by one form on the root box: every opaque
    (nonlinear) term is replaced by the end of its root-box interval that
    makes the row weakest, so any model of the form -- a point of the root
    box where it holds, without evaluation error -- satisfies the rows.  An
    equality with opaque terms relaxes to its two inequalities.  Returns a
    list of (rel, c0, symbol terms), [] when a needed interval is unbounded."""
    rel, c0, terms = form
    sym = {k: v for k, v in terms.items() if isinstance(k, str)}
    opq = [(k, v) for k, v in terms.items() if not isinstance(k, str)]
    if not opq:
        return [(rel, c0, sym)]
    lo_add = hi_add = 0
    for k, v in opq:
        lo, hi = ivl(k)
        if lo is None or hi is None:
            return []
        x, y = v * lo, v * hi
        lo_add += min(x, y)
        hi_add += max(x, y)
    if rel == 0:
        return [(0, c0 + lo_add, sym)]
    # sum == 0  ->  sym + c0 + lo_add <= 0  and  -(sym + c0 + hi_add) <= 0
    return [(0, c0 + lo_add, sym), (0, -(c0 + hi_add), {k: -v for k, v in sym.items()})]


def _emit_problem(var_names: List[str], lo: List[int], hi: List[int],
                  maximize: List[bool], atoms: List[Node]) -> Problem:
    if len(var_names) > MAX_VARS:
        raise CapacityError(f"{len(var_names)} free symbols in one component (> {MAX_VARS})")
    index = {n: i for i, n in enumerate(var_names)}
    em = _Emitter(index)
    # an atom that holds without error at every point of the root box (sound
    # interval proof, no possible EvalError) leaves the model set unchanged:
    # drop it (typically the far side of an overflow pin, x <= 2^63 - 1)
    ivl = _Ivl({n: (a, b) for n, a, b in zip(var_names, lo, hi)})
    atoms = [a for a in atoms
             if _may_err(a) or (_truth(a, ivl) != "T" and linear_truth(a, ivl) != "T")]
    # cheap linear rows first: a definitely-false atom ends evaluation early
    atoms = sorted(atoms, key=lambda a: (0 if a[0] == "p" and a[1] in ("le", "eq") else 1))
    for i, a in enumerate(atoms):
        em.atom(a, i)
    code, nregs, _ = em.finish([])
    if nregs - len(var_names) - len(em.consts) > MAX_TEMPS:
        raise CapacityError(f"search problem needs {nregs - len(var_names) - len(em.consts)} "
                            f"temporaries (> {MAX_TEMPS})")
    atom_regs = [0] * len(atoms)
    masks = []
    for a in atoms:
        m = 0
        for n in ir.symbols_of(a):
            m |= 1 << index[n]
        masks.append(m)
    # purely linear atoms double as contraction rows (sum <= 0 / sum == 0);
    # a disjunction of linear comparisons (and a linear !=, two strict
    # sides) becomes a row group the device contracts with whenever all but
    # one of its rows are infeasible on a box (include/mk_b200.h mk_row)
    rows: List[Tuple[int, int, List[Tuple[int, int]], int]] = []
    lin = _Lin({})
    group = 0
    seen_rows: Set[Tuple] = set()

    def add_row(rel: int, c0: int, terms: Dict[str, int], grp: int) -> None:
        key = (rel, c0, tuple(sorted(terms.items())), grp)
        if grp == 0 and key in seen_rows:
            return
        seen_rows.add(key)
        rows.append((rel, c0, [(index[k], v) for k, v in sorted(terms.items())], grp))

    for a in atoms:
        forms = _le_forms(lin, a) if a[0] == "p" else None
        if forms is not None and (a[1] != "ne" or not ROW_GROUPS):
            # a conjunct: its rows (opaque terms relaxed to their root-box
            # range) hold at every model
            if a[1] == "ne":
                continue
            for f in forms:
                for rel, c0, terms in _relax(f, ivl):
                    if terms:
                        add_row(rel, c0, terms, 0)
                    elif c0 > 0:
                        add_row(0, c0, {}, 0)         # no model: empty box
            continue
        if not ROW_GROUPS:
            continue
        ops = a[2] if a[0] == "o" and a[1] == "or" else (a,) if a[0] == "p" and a[1] == "ne" else ()
        alts = []
        for o in ops:
            got = _le_forms(lin, o)
            if got is None:
                alts = []
                break
            relaxed = []
            for f in got:
                r = _relax(f, ivl)
                if len(r) != 1:          # unbounded, or an equality with opaque terms
                    relaxed = None
                    break
                relaxed.append(r[0])
            if relaxed is None:
                alts = []
                break
            alts.extend(relaxed)
        # an alternative that holds on the whole box makes the group useless
        if len(alts) >= 2 and all(t or c0 > 0 for _, c0, t in alts):
            group += 1
            for rel, c0, terms in alts:
                add_row(rel, c0, terms, group)
    prob = Problem(var_names=var_names, lo=lo, hi=hi, maximize=maximize,
                   insns=code, consts=list(em.consts), nregs=nregs,
                   atom_regs=atom_regs, atom_masks=masks, rows=rows,
                   ops_per_point=len(code))
    prob.narrow = narrow_proof(prob)
    return prob


NARROW_LIMIT = 1 << 61
_I64_MIN, _I64_MAX = -(1 << 63), (1 << 63) - 1
_ARITH_CODES = frozenset({OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MOD, OP_EMOD, OP_SHL, OP_SHR})


def narrow_proof(p: Problem) -> bool:
    """True when exact 64-bit evaluation of ``p`` cannot overflow on the
    device (mk_core.cuh, MK_PF_NARROW).

    Runs the program once over the root box with interval bounds that
    contain the device's interval semantics (csrc/mk_core.cuh mk_iv_binop):
    every corner product of a multiplication is a product of in-range
    values, quotients are bounded by the dividend, remainders by the
    divisor.  Interval arithmetic is inclusion-isotonic, so the values the
    device computes on any sub-box or point lie inside these root ranges.
    Symbol bounds, arithmetic operands and results must stay inside
    (-2^61, 2^61); registers that are only compared (e.g. the i64 bounds of
    an overflow pin) need only fit in int64.  The contraction rows are
    bounded by the sum of |coef| * max|x| + |c0|."""
    nv = p.nvars
    R: Dict[int, Tuple[int, int]] = {}

    def small(r: Tuple[int, int]) -> bool:
        return -NARROW_LIMIT < r[0] and r[1] < NARROW_LIMIT

    for i in range(nv):
        R[i] = (p.lo[i], p.hi[i])
        if not small(R[i]):
            return False
    for j, c in enumerate(p.consts):
        if not _I64_MIN <= c <= _I64_MAX:
            return False
        R[nv + j] = (c, c)
    for op, d, a, b, c in p.insns:
        if op == OP_ATOM:
            continue
        A = R.get(a, (0, 0))
        B = R.get(b, (0, 0))
        if op in _ARITH_CODES and not (small(A) and small(B)):
            return False
        if op == OP_ADD:
            r = (A[0] + B[0], A[1] + B[1])
        elif op == OP_SUB:
            r = (A[0] - B[1], A[1] - B[0])
        elif op == OP_MUL:
            cs = (A[0] * B[0], A[0] * B[1], A[1] * B[0], A[1] * B[1])
            r = (min(cs), max(cs))
        elif op == OP_SHL:
            if B[0] != B[1] or B[0] < 0:
                return False
            r = (A[0] << B[0], A[1] << B[0])
        elif op == OP_SHR:
            if B[0] != B[1] or B[0] < 0:
                return False
            r = (A[0] >> B[0], A[1] >> B[0])
        elif op == OP_DIV:
            m = max(abs(A[0]), abs(A[1]))
            r = (-m, m)
        elif op == OP_MOD:
            m = max(abs(B[0]), abs(B[1]))
            r = (-m, m)
        elif op == OP_EMOD:
            r = (0, max(abs(B[0]), abs(B[1])))
        elif op == OP_ITE:
            C = R.get(c, (0, 0))
            r = (min(B[0], C[0]), max(B[1], C[1]))
        else:   # comparisons and booleans
            r = (0, 1)
        if op in _ARITH_CODES and not small(r):
            return False
        if not (_I64_MIN <= r[0] and r[1] <= _I64_MAX):
            return False
        R[d] = r
    for row in p.rows:
        c0, terms = row[1], row[2]
        s = abs(c0) + sum(abs(cf) * max(abs(p.lo[v]), abs(p.hi[v])) for v, cf in terms)
        if s >= NARROW_LIMIT:
            return False
    return True


# -- driver ------------------------------------------------------------------------------

def _components(assertions: Sequence[Node]) -> List[List[Node]]:
    """Union-find over shared symbols, symbol-free assertions ride with the
    first group (solver/builtin.py:767-793)."""
    parent = list(range(len(assertions)))

    def find(i: int) -> int:
        while parent[i] != i:
            parent[i] = parent[parent[i]]
            i = parent[i]
        return i

    owner: Dict[str, int] = {}
    for i, a in enumerate(assertions):
        for name in ir.symbols_of(a):
            if name in owner:
                parent[find(i)] = find(owner[name])
            else:
                owner[name] = i
    groups: Dict[int, List[Node]] = {}
    order: List[int] = []
    for i, a in enumerate(assertions):
        r = find(i)
        if r not in groups:
            groups[r] = []
            order.append(r)
        groups[r].append(a)
    return [groups[r] for r in order]


def _emit_component(ps: "_Presolve", problems: List[Problem]) -> List[int]:
    """Independent device problems of one presolved component (its atoms
    split over shared free symbols); appended to ``problems``, indices
    returned."""
    out: List[int] = []
    free = [n for n in ps.bounds]
    atom_vars = [set(ir.symbols_of(a)) for a in ps.atoms]
    parent = {n: n for n in free}

    def find(x: str) -> str:
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for vs in atom_vars:
        vs = list(vs)
        for o in vs[1:]:
            ra, rb = find(vs[0]), find(o)
            if ra != rb:
                parent[ra] = rb
    buckets: Dict[str, List[int]] = {}
    for i, vs in enumerate(atom_vars):
        if vs:
            buckets.setdefault(find(next(iter(vs))), []).append(i)
    used: Set[str] = set()
    for root, idxs in buckets.items():
        names = sorted({n for i in idxs for n in atom_vars[i]}, key=lambda n: ps.pos[n])
        used |= set(names)
        lo = [ps.bounds[n][0] for n in names]
        hi = [ps.bounds[n][1] for n in names]
        if any(v is None for v in lo + hi):
            raise CapacityError("unbounded free symbol after presolve")
        mx = [ps.maximize.get(n, False) for n in names]
        out.append(len(problems))
        problems.append(_emit_problem(names, lo, hi, mx, [ps.atoms[i] for i in idxs]))
    # free symbols constrained by bounds only: their optimum is a bound,
    # still decided on the device as an atom-free problem
    rest = sorted((n for n in free if n not in used), key=lambda n: ps.pos[n])
    if rest:
        lo = [ps.bounds[n][0] for n in rest]
        hi = [ps.bounds[n][1] for n in rest]
        if any(v is None for v in lo + hi):
            raise CapacityError("unbounded free symbol after presolve")
        mx = [ps.maximize.get(n, False) for n in rest]
        out.append(len(problems))
        problems.append(_emit_problem(rest, lo, hi, mx, []))
    return out


def _split_disjunction(ps: "_Presolve"):
    """Case split on one disjunction left after presolve, as the reference
    expands boolean paths (solver/linear.py:313-372): the component's models
    are the union over the disjuncts of the models of (rest and disjunct).
    Each branch is presolved on its own.  One surviving branch IS the
    component (same model set, so the same canonical witness); two or more
    come back as a list: the device searches each branch (its disjunct is a
    linear row there, where the disjunction left only interval splitting)
    and the component's witness is the best branch optimum in witness order
    (CompiledQuery.assemble)."""
    for a in ps.atoms:
        if a[0] == "o" and a[1] == "or" and 2 <= len(a[2]) <= 4:
            break
    else:
        return ps
    rest = [x for x in ps.atoms if x is not a]
    live = []
    for d in a[2]:
        f = ps.fork(rest + [d])
        try:
            f.run()
        except CompileError:
            return ps
        if not f.unsat:
            live.append(f)
    if not live:
        ps.unsat = True
        return ps
    return live[0] if len(live) == 1 else live


def compile_query(assertions: Sequence[Node],
                  origin_of: Callable[[str], str], light: bool = False) -> CompiledQuery:
    """Compile one checker query (a list of IR assertions); ``light``: the
    structural presolve only (_Presolve.light)."""
    with ir.compile_scope():
        return _compile_query(assertions, origin_of, light)


def _compile_query(assertions: Sequence[Node],
                   origin_of: Callable[[str], str], light: bool = False) -> CompiledQuery:
    widths: Dict[str, str] = {}
    for a in assertions:
        ir.symbols_of(a, widths)
    order = optimization_order(widths, origin_of)
    pos = {n: float(i) for i, (n, _) in enumerate(order)}
    maximize = {n: d == "max" for n, d in order}
    witness_names = sorted(widths)

    simplified = [ir.simplify(a) for a in assertions]
    groups: List[Group] = []
    problems: List[Problem] = []
    defs: Dict[str, Node] = {}
    free_default: Dict[str, int] = {}
    seen_syms: Set[str] = set()

    entailed = refmirror.entailed_bounds(simplified)
    for comp in _components(simplified):
        csyms: Dict[str, str] = {}
        for a in comp:
            ir.symbols_of(a, csyms)
        seen_syms |= set(csyms)
        # the reference gives up on the whole component when its division
        # rewrite or path expansion raises (solver/builtin.py:805-811)
        reason = refmirror.component_giveup(comp, entailed)
        if reason:
            groups.append(Group("unknown", reason, True))
            continue
        flags = {"unsupported": False}
        try:
            atoms = [ir.simplify(_nnf(a, False, flags)) for a in comp]
            # the reference's division rewrite adds its case split for a
            # symbolic divisor as a top-level side constraint, so no model of
            # the component has a zero divisor anywhere, even inside an
            # operand a short-circuit would skip (solver/linear.py:5-10,
            # :184-259)
            atoms.extend(("p", "ne", d, ("c", 0, ir.width_of(d))) for d in _symbolic_divisors(comp))
        except CompileError as exc:
            groups.append(Group("unknown", str(exc), True))
            continue
        int_widths = {n: w for n, w in csyms.items() if not ir.is_float(w)}
        ps = _Presolve(atoms, dict(int_widths), dict(pos), dict(maximize), light)
        try:
            ps.run()
        except CompileError as exc:
            groups.append(Group("unknown", str(exc), True))
            continue
        had = flags["unsupported"]
        if not ps.unsat and OR_SPLIT and not light:
            ps = _split_disjunction(ps)
        if not isinstance(ps, list) and ps.unsat:
            if not had:
                # one unsatisfiable component refutes the query whatever the
                # others are (solver/builtin.py:737-740): nothing of it goes
                # to the device, and the remaining components are not compiled
                return CompiledQuery(witness_names=witness_names, order=order,
                                     groups=[Group("unsat", "presolve", False)], problems=[],
                                     defs={}, free_default={})
            groups.append(Group("unknown", "float/unsupported atoms only", had))
            continue
        if isinstance(ps, list):
            # live disjunct branches: each its own problems and definitions;
            # the component's models are their union (Group.alts)
            grp = Group("pending", None, had)
            for f in ps:
                idx = _emit_component(f, problems)
                grp.alts.append((idx, dict(f.defs), sorted(csyms)))
            groups.append(grp)
            continue
        for n, e in ps.defs.items():
            defs[n] = e
        grp = Group("pending", None, had)
        grp.problems.extend(_emit_component(ps, problems))
        groups.append(grp)

    if any(g.status == "unknown" for g in groups):
        # the verdict is unknown unless another component is unsat
        # (solver/builtin.py:737-745): the device only needs feasibility
        for p in problems:
            p.any_model = True
    # symbols that simplification removed entirely: unconstrained, so the
    # canonical value is the width bound in the optimisation direction
    for n, w in widths.items():
        if n not in seen_syms and not ir.is_float(w):
            lo, hi = ir.bounds(w)
            free_default[n] = hi if maximize.get(n) else lo
    return CompiledQuery(witness_names=witness_names, order=order, groups=groups,
                         problems=problems, defs=defs, free_default=free_default)
