"""Mirror of the reference solver's *structural* give-ups.

The reference decides a component with ``_check_component``
(solver/builtin.py:796-843), which first eliminates div/mod/emod/shr
(``rewrite_divs``, solver/linear.py:130-306) and expands the boolean structure
into paths (``boolean_paths``, solver/linear.py:313-372).  Either step can
raise: an unsupported construct, or more than ``max_paths`` (512,
solver/interface.py:27) case splits.  The component is then ``unknown``
whatever its models are, and so is the site (unless another component is
unsat, solver/builtin.py:737-750).

To return the reference's verdict on such sites the compiler asks
:func:`component_giveup` first.  This module restates exactly the parts of
those two functions that decide *whether* they raise: the sign-case structure
of the division rewrite (which depends on the reference's interval analysis,
restated here as :func:`ref_interval`) and the path-expansion traversal with
its cap check.  It builds no linear systems.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

from . import ir
from .ir import Node

Interval = Tuple[Optional[int], Optional[int]]
FULL: Interval = (None, None)
I64_BOUNDS = ir.bounds("i64")


class GiveUp(Exception):
    """The reference raises Unsupported / CapExceeded for this component."""


# -- sym/expr.py:676-752 -----------------------------------------------------------

def _add_b(a, b):
    return None if a is None or b is None else a + b


def _neg_b(a):
    return None if a is None else -a


def _mul_candidates(x: Interval, y: Interval) -> Interval:
    cands = []
    for a in x:
        for b in y:
            if a is None or b is None:
                return FULL
            cands.append(a * b)
    return (min(cands), max(cands))


def _tdiv(a: int, b: int) -> int:
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def ref_interval(e: Node, bounds: Dict[str, Interval]) -> Interval:
    """The reference's conservative range (sym/expr.py:676-752), restated
    operator by operator so case decisions match it exactly."""

    def go(e: Node) -> Interval:
        t = e[0]
        w = ir.width_of(e)
        if ir.is_float(w) and t not in ("p", "o"):
            return FULL
        if t == "c":
            return (e[1], e[1]) if isinstance(e[1], int) else FULL
        if t == "s":
            got = bounds.get(e[1])
            if got is not None:
                return got
            return ir.bounds(e[2])
        if t in ("p", "o"):
            return (0, 1)
        if t == "x":
            if ir.is_float(e[2]) or ir.is_float(ir.width_of(e[1])):
                return FULL
            return go(e[1])
        if t == "i":
            lt, lo_ = go(e[2]), go(e[3])
            lo = None if lt[0] is None or lo_[0] is None else min(lt[0], lo_[0])
            hi = None if lt[1] is None or lo_[1] is None else max(lt[1], lo_[1])
            return (lo, hi)
        op = e[1]
        x, y = go(e[2]), go(e[3])
        rhs = e[3]
        if op == "add":
            return (_add_b(x[0], y[0]), _add_b(x[1], y[1]))
        if op == "sub":
            return (_add_b(x[0], _neg_b(y[1])), _add_b(x[1], _neg_b(y[0])))
        if op == "mul":
            return _mul_candidates(x, y)
        if op == "div":
            if y[0] is not None and y[0] >= 1 or y[1] is not None and y[1] <= -1:
                cands = []
                for a in x:
                    for b in y:
                        if a is None or b is None:
                            return FULL
                        cands.append(_tdiv(a, b))
                return (min(cands), max(cands))
            return FULL
        if op == "mod":
            if rhs[0] == "c" and rhs[1] != 0:
                m = abs(rhs[1]) - 1
                lo = 0 if (x[0] is not None and x[0] >= 0) else -m
                hi = 0 if (x[1] is not None and x[1] <= 0) else m
                return (lo, hi)
            return FULL
        if op == "emod":
            if rhs[0] == "c" and rhs[1] != 0:
                return (0, abs(rhs[1]) - 1)
            return (0, None)
        if op == "shl":
            if rhs[0] == "c" and 0 <= rhs[1] <= 256:
                f = 1 << rhs[1]
                return _mul_candidates(x, (f, f))
            return FULL
        if op == "shr":
            if rhs[0] == "c" and 0 <= rhs[1] <= 256:
                lo = None if x[0] is None else x[0] >> rhs[1]
                hi = None if x[1] is None else x[1] >> rhs[1]
                return (lo, hi)
            return FULL
        raise AssertionError(op)

    return go(e)


# -- solver/builtin.py:657-702 ---------------------------------------------------------

_FLIPC = {"lt": "gt", "le": "ge", "gt": "lt", "ge": "le", "eq": "eq"}


def entailed_bounds(assertions: Sequence[Node]) -> Dict[str, Interval]:
    out: Dict[str, Interval] = {}

    def tighten(name, lo, hi):
        blo, bhi = out.get(name, (None, None))
        if lo is not None:
            blo = lo if blo is None else max(blo, lo)
        if hi is not None:
            bhi = hi if bhi is None else min(bhi, hi)
        out[name] = (blo, bhi)

    stack = list(assertions)
    while stack:
        e = stack.pop()
        if e[0] == "o" and e[1] == "and":
            stack.extend(e[2])
            continue
        if e[0] != "p":
            continue
        lhs, rhs, op = e[2], e[3], e[1]
        if lhs[0] == "c" and rhs[0] == "s":
            lhs, rhs, op = rhs, lhs, _FLIPC.get(op, op)
        if not (lhs[0] == "s" and rhs[0] == "c"):
            continue
        if ir.is_float(lhs[2]) or not isinstance(rhs[1], int):
            continue
        v = rhs[1]
        if op == "eq":
            tighten(lhs[1], v, v)
        elif op == "le":
            tighten(lhs[1], None, v)
        elif op == "lt":
            tighten(lhs[1], None, v - 1)
        elif op == "ge":
            tighten(lhs[1], v, None)
        elif op == "gt":
            tighten(lhs[1], v + 1, None)
    return out


# -- solver/linear.py:130-306 (case structure only) -------------------------------------

def _c(v: int, w: str) -> Node:
    return ("c", v, w)


def rewrite_divs(assertions: Sequence[Node], bounds: Dict[str, Interval]) -> List[Node]:
    """Rewritten assertions plus side constraints, with the same boolean
    shape as the reference's (fresh symbols named like its ``_Fresh``)."""
    counter = [0]
    sides: List[Node] = []
    bmap: Dict[str, Interval] = dict(bounds)

    def fresh(prefix: str, w: str) -> Node:
        s = ("s", f"${prefix}{counter[0]}", w)
        counter[0] += 1
        return s

    def iv(e: Node) -> Interval:
        return ref_interval(e, bmap)

    def record(sym: Node, lo, hi) -> None:
        bmap[sym[1]] = (lo, hi)

    def cmp(op, a, b):
        return ("p", op, a, b)

    def bop(op, a, b, w):
        return ("b", op, a, b, w)

    def div_by_const(x: Node, c: int, w: str) -> Node:
        if c == 0:
            raise GiveUp("unsupported: division by constant zero")
        if c < 0:
            inner = div_by_const(x, -c, w)
            return bop("sub", _c(0, w), inner, w)
        q = fresh("q", w)
        xlo, xhi = iv(x)
        record(q, None if xlo is None else _tdiv(xlo, c) - 1,
               None if xhi is None else _tdiv(xhi, c) + 1)
        r = bop("sub", x, bop("mul", q, _c(c, w), w), w)
        nonneg = ("o", "and", (cmp("ge", r, _c(0, w)), cmp("le", r, _c(c - 1, w))))
        nonpos = ("o", "and", (cmp("le", r, _c(0, w)), cmp("ge", r, _c(1 - c, w))))
        if xlo is not None and xlo >= 0:
            sides.append(nonneg)
        elif xhi is not None and xhi <= 0:
            sides.append(nonpos)
        else:
            sides.append(("o", "or", (("o", "and", (cmp("ge", x, _c(0, w)), nonneg)),
                                      ("o", "and", (cmp("le", x, _c(0, w)), nonpos)))))
        return q

    def div_by_sym(x: Node, d: Node, w: str) -> Node:
        q = fresh("q", w)
        record(q, *I64_BOUNDS)
        r = bop("sub", x, bop("mul", d, q, w), w)
        dlo, dhi = iv(d)
        xlo, xhi = iv(x)
        d_cases = []
        if dhi is None or dhi >= 1:
            d_cases.append((cmp("ge", d, _c(1, w)), bop("sub", d, _c(1, w), w)))
        if dlo is None or dlo <= -1:
            nd = bop("sub", _c(0, w), d, w)
            d_cases.append((cmp("le", d, _c(-1, w)), bop("sub", nd, _c(1, w), w)))
        if not d_cases:
            raise GiveUp("unsupported: divisor has empty sign range")
        x_cases = []
        if xhi is None or xhi >= 0:
            x_cases.append((cmp("ge", x, _c(0, w)), "nonneg"))
        if xlo is None or xlo < 0:
            x_cases.append((cmp("le", x, _c(0, w)), "nonpos"))
        alts = []
        for dcond, dm1 in d_cases:
            for xcond, kind in x_cases:
                if kind == "nonneg":
                    body = ("o", "and", (cmp("ge", r, _c(0, w)), cmp("le", r, dm1)))
                else:
                    neg_dm1 = bop("sub", _c(0, w), dm1, w)
                    body = ("o", "and", (cmp("le", r, _c(0, w)), cmp("ge", r, neg_dm1)))
                alts.append(("o", "and", (dcond, xcond, body)))
        sides.append(alts[0] if len(alts) == 1 else ("o", "or", tuple(alts)))
        return q

    def emod(x: Node, d: Node, w: str) -> Node:
        r = fresh("r", w)
        k = fresh("k", w)
        record(k, *I64_BOUNDS)
        prod = bop("mul", d, k, w) if d[0] != "c" else bop("mul", k, d, w)
        sides.append(cmp("eq", bop("sub", x, r, w), prod))
        sides.append(cmp("ge", r, _c(0, w)))
        if d[0] == "c":
            if d[1] == 0:
                raise GiveUp("unsupported: emod by constant zero")
            record(r, 0, abs(d[1]) - 1)
            sides.append(cmp("le", r, _c(abs(d[1]) - 1, w)))
        else:
            record(r, 0, None)
            dlo, dhi = iv(d)
            alts = []
            if dhi is None or dhi >= 1:
                alts.append(("o", "and", (cmp("ge", d, _c(1, w)),
                                          cmp("le", r, bop("sub", d, _c(1, w), w)))))
            if dlo is None or dlo <= -1:
                nd = bop("sub", _c(0, w), d, w)
                alts.append(("o", "and", (cmp("le", d, _c(-1, w)),
                                          cmp("le", r, bop("sub", nd, _c(1, w), w)))))
            if not alts:
                raise GiveUp("unsupported: emod divisor has empty sign range")
            sides.append(alts[0] if len(alts) == 1 else ("o", "or", tuple(alts)))
        return r

    def floor_pow2(x: Node, c: int, w: str) -> Node:
        m = 1 << c
        q = fresh("q", w)
        xlo, xhi = iv(x)
        record(q, None if xlo is None else xlo >> c, None if xhi is None else xhi >> c)
        r = bop("sub", x, bop("mul", q, _c(m, w), w), w)
        sides.append(cmp("ge", r, _c(0, w)))
        sides.append(cmp("le", r, _c(m - 1, w)))
        return q

    def go(e: Node) -> Node:
        kids = ir.children(e)
        if kids:
            new = tuple(go(c) for c in kids)
            if new != kids:
                e = ir.rebuild(e, new)
        if e[0] != "b":
            return e
        op, lhs, rhs, w = e[1], e[2], e[3], e[4]
        if op == "div":
            if rhs[0] == "c":
                return div_by_const(lhs, rhs[1], w)
            return div_by_sym(lhs, rhs, w)
        if op == "mod":
            if rhs[0] == "c":
                q = div_by_const(lhs, rhs[1], w)
                return bop("sub", lhs, bop("mul", q, _c(rhs[1], w), w), w)
            q = div_by_sym(lhs, rhs, w)
            return bop("sub", lhs, bop("mul", rhs, q, w), w)
        if op == "emod":
            return emod(lhs, rhs, w)
        if op == "shr":
            if rhs[0] != "c" or not (0 <= rhs[1] <= 256):
                raise GiveUp("unsupported: shift amount must be a small constant")
            return floor_pow2(lhs, rhs[1], w)
        return e

    out = [go(a) for a in assertions]
    out.extend(sides)
    return out


# -- solver/linear.py:65-105, 313-372 ------------------------------------------------------

_NEGC = {"eq": "ne", "ne": "eq", "lt": "ge", "le": "gt", "gt": "le", "ge": "lt"}


def _negate(e: Node) -> Node:
    t = e[0]
    if t == "c":
        return ("c", 0 if e[1] else 1, "bool")
    if t == "p":
        return ("p", _NEGC[e[1]], e[2], e[3])
    if t == "o":
        if e[1] == "not":
            return e[2][0]
        flipped = "or" if e[1] == "and" else "and"
        return ("o", flipped, tuple(_negate(a) for a in e[2]))
    if t == "i":
        return ("i", e[1], _negate(e[2]), _negate(e[3]), "bool")
    if t == "s" and e[2] == "bool":
        return ("p", "eq", e, ("c", 0, "bool"))
    raise GiveUp(f"unsupported: cannot negate {t}")


def _find_int_ite(e: Node) -> Optional[Node]:
    scope = ir.CompileScope._active
    if scope is None:
        return _find_int_ite_walk(e)
    key = ("int_ite", e)
    if key in scope.extra:
        return scope.extra[key]
    got = _find_int_ite_walk(e)
    scope.extra[key] = got
    return got


def _find_int_ite_walk(e: Node) -> Optional[Node]:
    if e[0] == "i" and e[4] != "bool":
        return e
    for c in ir.children(e):
        got = _find_int_ite(c)
        if got is not None:
            return got
    return None


def _find_any_ite(e: Node) -> bool:
    if e[0] == "i":
        return True
    return any(_find_any_ite(c) for c in ir.children(e))


def _replace_all(e: Node, old: Node, new: Node) -> Node:
    if e == old:
        return new
    kids = ir.children(e)
    if not kids:
        return e
    repl = tuple(_replace_all(c, old, new) for c in kids)
    return e if repl == kids else ir.rebuild(e, repl)


def count_paths(assertions: Sequence[Node], cap: int) -> int:
    """Restates boolean_paths' traversal and cap check; returns the number of
    surviving paths or raises GiveUp exactly when the reference raises.

    Pending conjunct lists are persistent cons lists ((head, tail) pairs,
    None at the end): the reference's ``[x] + pending`` prepends and
    ``pending.pop(0)`` become O(1) while the traversal order, and so every
    ``len(work) + done > cap`` check, is unchanged."""
    done = 0
    pend0 = None
    for a in reversed(list(assertions)):
        pend0 = (a, pend0)
    work: List[object] = [pend0]
    simp: Dict[Node, Node] = {}
    # integer if-then-else never appears unless the input has one
    has_ite = any(_find_any_ite(a) for a in assertions)
    while work:
        if len(work) + done > cap:
            raise GiveUp(f"more than {cap} case splits")
        pending = work.pop()
        alive = True
        while pending is not None:
            raw, pending = pending
            e = simp.get(raw)
            if e is None:
                e = ir.simplify(raw)
                simp[raw] = e
            t = e[0]
            if t == "c":
                if e[2] != "bool":
                    raise GiveUp("unsupported: non-boolean assertion")
                if e[1]:
                    continue
                alive = False
                break
            if t == "o":
                if e[1] == "and":
                    for arm in reversed(e[2]):
                        pending = (arm, pending)
                    continue
                if e[1] == "not":
                    pending = (_negate(e[2][0]), pending)
                    continue
                for arm in reversed(e[2]):
                    work.append((arm, pending))
                alive = False
                break
            if t == "i":
                work.append((_negate(e[1]), (e[3], pending)))
                work.append((e[1], (e[2], pending)))
                alive = False
                break
            if t == "s":
                if e[2] != "bool":
                    raise GiveUp("unsupported: non-boolean assertion")
                continue
            if t == "p":
                ite = _find_int_ite(e) if has_ite else None
                if ite is not None:
                    then_atom = _replace_all(e, ite, ite[2])
                    else_atom = _replace_all(e, ite, ite[3])
                    work.append((_negate(ite[1]), (else_atom, pending)))
                    work.append((ite[1], (then_atom, pending)))
                    alive = False
                    break
                if e[1] == "ne":
                    work.append((("p", "gt", e[2], e[3]), pending))
                    work.append((("p", "lt", e[2], e[3]), pending))
                    alive = False
                    break
                continue
            raise GiveUp(f"unsupported: cannot assert a {t}")
        if alive:
            done += 1
    return done


def _path_bound(e: Node, neg: bool, cap: int) -> int:
    """Upper bound on the paths boolean_paths expands ``e`` (or its negation)
    into; every pending work item stands for at least one of them, so
    ``len(work) + done`` never exceeds this bound.  Saturates at cap + 1."""
    t = e[0]
    if t == "o":
        if e[1] == "not":
            return _path_bound(e[2][0], not neg, cap)
        conj = (e[1] == "and") != neg
        acc = 1 if conj else 0
        for a in e[2]:
            b = _path_bound(a, neg, cap)
            acc = acc * b if conj else acc + b
            if acc > cap:
                return cap + 1
        return max(acc, 1)
    if t == "p":
        if _find_int_ite(e) is not None:
            return cap + 1
        op = _NEGC[e[1]] if neg else e[1]
        return 2 if op == "ne" else 1
    if t == "i":
        return cap + 1
    return 1


class _NoCount(Exception):
    pass


def _live(e: Node, cap: int, simp: Dict[Node, Node]) -> int:
    """Number of live paths boolean_paths' traversal completes for the one
    conjunct ``e`` (simplify is context-free, so a dead alternative is dead
    in every combination and counts multiply / add); saturates at cap + 2.
    Forms the traversal would raise on, or integer if-then-else, are not
    counted (_NoCount)."""
    top = cap + 2
    r = simp.get(e)
    if r is None:
        r = ir.simplify(e)
        simp[e] = r
    t = r[0]
    if t == "c":
        if r[2] != "bool":
            raise _NoCount()
        return 1 if r[1] else 0
    if t == "s":
        if r[2] != "bool":
            raise _NoCount()
        return 1
    if t == "o":
        if r[1] == "not":
            try:
                return _live(_negate(r[2][0]), cap, simp)
            except GiveUp:
                raise _NoCount()
        if r[1] == "and":
            acc = 1
            for a in r[2]:
                acc = min(top, acc * _live(a, cap, simp))
                if acc == 0:
                    return 0
            return acc
        acc = 0
        for a in r[2]:
            acc = min(top, acc + _live(a, cap, simp))
        return acc
    if t == "i":
        try:
            nc = _negate(r[1])
        except GiveUp:
            raise _NoCount()
        a = min(top, _live(r[1], cap, simp) * _live(r[2], cap, simp))
        b = min(top, _live(nc, cap, simp) * _live(r[3], cap, simp))
        return min(top, a + b)
    if t == "p":
        if _find_int_ite(r) is not None:
            raise _NoCount()
        if r[1] == "ne":
            return min(top, _live(("p", "gt", r[2], r[3]), cap, simp)
                       + _live(("p", "lt", r[2], r[3]), cap, simp))
        return 1
    raise _NoCount()


def live_paths(assertions: Sequence[Node], cap: int) -> Optional[int]:
    """Exact number of paths boolean_paths completes (saturated at cap + 2),
    or None when the traversal must run (forms it raises on, int ite)."""
    simp: Dict[Node, Node] = {}
    acc = 1
    try:
        for a in assertions:
            acc = min(cap + 2, acc * _live(a, cap, simp))
            if acc == 0:
                return 0
    except _NoCount:
        return None
    return acc


def component_giveup(component: Sequence[Node], bounds: Dict[str, Interval],
                     max_paths: int = 512) -> Optional[str]:
    """The reason the reference gives up on this (simplified) component in
    solver/builtin.py:805-811, or None when it proceeds to linearisation."""
    try:
        rewritten = rewrite_divs(component, bounds)
        total = 1
        for a in rewritten:
            total *= _path_bound(a, False, max_paths)
            if total > max_paths:
                break
        if total > max_paths:
            # at least cap + 2 live paths: the traversal's check
            # len(work) + done > cap fires for certain (after the (cap+1)-th
            # completed path a live one is still pending); otherwise (or when
            # the count does not apply) the exact traversal decides
            live = live_paths(rewritten, max_paths)
            if live is not None and live >= max_paths + 2:
                raise GiveUp(f"more than {max_paths} case splits")
            count_paths(rewritten, max_paths)   # exact traversal only when needed
    except GiveUp as g:
        return str(g)
    return None
