"""Host-side expression IR for site queries.

A site query is a list of boolean assertions over named integer symbols.
This module holds a compact, hashable tuple form of the reference's
expression algebra (``minikernel/sym/expr.py``) so the site compiler can
work without importing the reference, plus the conversions to and from
the reference's objects and a JSON wire form used by the golden fixtures.

Node layouts (all plain tuples, so structural equality and hashing are free):

    ('c', value, width)              constant   (reference Const, sym/expr.py:123-142)
    ('s', name, width)               symbol     (Sym, sym/expr.py:145-150)
    ('b', op, lhs, rhs, width)       arithmetic (BinOp, sym/expr.py:153-162)
    ('x', arg, width)                cast       (Cast, sym/expr.py:165-171)
    ('p', op, lhs, rhs)              compare    (Cmp, sym/expr.py:174-186)
    ('o', op, args)                  and/or/not (BoolOp, sym/expr.py:189-203)
    ('i', cond, then, other, width)  if-then-else (Ite, sym/expr.py:206-211)

Widths are the reference's width names ('bool', 'i32', 'u64', 'f32', ...).

Semantics are the reference's *mathematical* mode: unbounded integers,
integer casts are the identity, truncating div/mod, Euclidean emod,
``shl`` = multiply by 2^k, ``shr`` = floor shift (sym/expr.py:273-383).
"""

from __future__ import annotations

from fractions import Fraction
from typing import Dict, Iterable, List, Mapping, Optional, Sequence, Tuple

Node = tuple

# -- widths ------------------------------------------------------------------

_WIDTH_INFO = {
    # name: (bits, signed, is_float)
    "bool": (1, False, False),
    "i16": (16, True, False),
    "u16": (16, False, False),
    "i32": (32, True, False),
    "u32": (32, False, False),
    "i64": (64, True, False),
    "u64": (64, False, False),
    "f16": (16, True, True),
    "f32": (32, True, True),
    "f64": (64, True, True),
}

ARITH_OPS = frozenset({"add", "sub", "mul", "div", "mod", "emod", "shl", "shr"})
CMP_OPS = frozenset({"eq", "ne", "lt", "le", "gt", "ge"})
BOOL_OPS = frozenset({"and", "or", "not"})
_WRAP_HOM_OPS = frozenset({"add", "sub", "mul"})  # sym/expr.py:92


def is_float(w: str) -> bool:
    return _WIDTH_INFO[w][2]


def bits(w: str) -> int:
    return _WIDTH_INFO[w][0]


def bounds(w: str) -> Tuple[int, int]:
    """Inclusive integer range of a width (sym/expr.py:57-66)."""
    b, signed, flt = _WIDTH_INFO[w]
    if flt:
        raise ValueError("float widths have no integer bounds")
    if b == 1:
        return (0, 1)
    if signed:
        half = 1 << (b - 1)
        return (-half, half - 1)
    return (0, (1 << b) - 1)


class EvalError(ValueError):
    """Evaluation failed: division by zero or a malformed shift
    (sym/expr.py:29-30).  A point that raises is not a model."""


# -- constructors --------------------------------------------------------------

def const(v, w: str) -> Node:
    if is_float(w):
        return ("c", Fraction(v), w)
    return ("c", int(v), w)


def sym(name: str, w: str) -> Node:
    return ("s", name, w)


TRUE = ("c", 1, "bool")
FALSE = ("c", 0, "bool")


def width_of(e: Node) -> str:
    t = e[0]
    if t in ("c", "s"):
        return e[2]
    if t == "b":
        return e[4]
    if t == "x":
        return e[2]
    if t in ("p", "o"):
        return "bool"
    if t == "i":
        return e[4]
    raise TypeError(f"not an IR node: {e!r}")


def children(e: Node) -> Tuple[Node, ...]:
    t = e[0]
    if t in ("c", "s"):
        return ()
    if t in ("b", "p"):
        return (e[2], e[3])
    if t == "x":
        return (e[1],)
    if t == "o":
        return e[2]
    if t == "i":
        return (e[1], e[2], e[3])
    raise TypeError(f"not an IR node: {e!r}")


def rebuild(e: Node, kids: Sequence[Node]) -> Node:
    t = e[0]
    if t in ("c", "s"):
        return e
    if t == "b":
        return ("b", e[1], kids[0], kids[1], e[4])
    if t == "p":
        return ("p", e[1], kids[0], kids[1])
    if t == "x":
        return ("x", kids[0], e[2])
    if t == "o":
        return ("o", e[1], tuple(kids))
    if t == "i":
        return ("i", kids[0], kids[1], kids[2], e[4])
    raise TypeError(f"not an IR node: {e!r}")


def and_(*args: Node) -> Node:
    """sym/expr.py:222-232"""
    flat = [a for a in args if a != TRUE]
    if not flat:
        return TRUE
    if len(flat) == 1:
        return flat[0]
    return ("o", "and", tuple(flat))


def not_(a: Node) -> Node:
    return ("o", "not", (a,))


# -- traversal -------------------------------------------------------------------

class CompileScope:
    """Memo tables shared by every simplify / symbols_of call inside one site
    compilation (``with ir.compile_scope(): ...``).  Both functions are pure,
    so sharing within a query is exact; the scope ends with the query, so
    nothing is reused across queries or calls."""

    _active: Optional["CompileScope"] = None

    def __init__(self) -> None:
        self.simplify: Dict[Node, Node] = {}
        self.symbols: Dict[Node, Tuple[Tuple[str, str], ...]] = {}
        self.extra: Dict[Tuple, object] = {}     # other pure per-node helpers

    def __enter__(self) -> "CompileScope":
        self._prev = CompileScope._active
        CompileScope._active = self
        return self

    def __exit__(self, *exc) -> None:
        CompileScope._active = self._prev


def compile_scope() -> CompileScope:
    return CompileScope()


def symbols_of(e: Node, out: Optional[Dict[str, str]] = None) -> Dict[str, str]:
    """name -> width, first-occurrence order (sym/expr.py:390-402)."""
    if out is None:
        out = {}
    scope = CompileScope._active
    if scope is not None:
        got = scope.symbols.get(e)
        if got is None:
            got = tuple(_symbols_walk(e, {}).items())
            scope.symbols[e] = got
        for n, w in got:
            if n not in out:
                out[n] = w
        return out
    return _symbols_walk(e, out)


def _symbols_walk(e: Node, out: Dict[str, str]) -> Dict[str, str]:
    stack = [e]
    # iterative pre-order keeping left-to-right first occurrence
    while stack:
        n = stack.pop()
        if n[0] == "s":
            if n[1] not in out:
                out[n[1]] = n[2]
            continue
        kids = children(n)
        for k in reversed(kids):
            stack.append(k)
    return out


def contains(e: Node, needle: Node) -> bool:
    if e == needle:
        return True
    return any(contains(c, needle) for c in children(e))


def substitute(e: Node, mapping: Mapping[str, Node],
               memo: Optional[Dict[Node, Node]] = None) -> Node:
    """``e`` with every symbol of ``mapping`` replaced; ``memo`` may be shared
    by calls with the same mapping (shared subtrees are rewritten once)."""
    if not mapping:
        return e
    if memo is None:
        memo = {}

    def go(n: Node) -> Node:
        got = memo.get(n)
        if got is not None:
            return got
        if n[0] == "s":
            r = mapping.get(n[1], n)
        else:
            kids = children(n)
            if not kids:
                r = n
            else:
                new = tuple(go(c) for c in kids)
                r = n if new == kids else rebuild(n, new)
        memo[n] = r
        return r

    return go(e)


# -- evaluation (mathematical mode) ---------------------------------------------------

def _trunc_div(a, b):
    """sym/expr.py:273-279"""
    if b == 0:
        raise EvalError("division by zero")
    if isinstance(a, Fraction) or isinstance(b, Fraction):
        return Fraction(a) / Fraction(b)
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def _trunc_mod(a: int, b: int) -> int:
    """sym/expr.py:282-285"""
    if b == 0:
        raise EvalError("remainder by zero")
    return a - _trunc_div(a, b) * b


def _euclid_mod(a: int, b: int) -> int:
    """sym/expr.py:288-291"""
    if b == 0:
        raise EvalError("remainder by zero")
    return a % abs(b)


def _shift_amount(b) -> int:
    """sym/expr.py:294-299"""
    if not isinstance(b, int) or b < 0:
        raise EvalError(f"bad shift amount: {b}")
    if b > (1 << 20):
        raise EvalError(f"shift amount too large: {b}")
    return b


def apply_binop(op: str, a, b):
    """sym/expr.py:302-319"""
    if op == "add":
        return a + b
    if op == "sub":
        return a - b
    if op == "mul":
        return a * b
    if op == "div":
        return _trunc_div(a, b)
    if op == "mod":
        return _trunc_mod(a, b)
    if op == "emod":
        return _euclid_mod(a, b)
    if op == "shl":
        return a * (1 << _shift_amount(b))
    if op == "shr":
        return a >> _shift_amount(b)
    raise AssertionError(op)


_CMP = {
    "eq": lambda a, b: a == b,
    "ne": lambda a, b: a != b,
    "lt": lambda a, b: a < b,
    "le": lambda a, b: a <= b,
    "gt": lambda a, b: a > b,
    "ge": lambda a, b: a >= b,
}


def evaluate(e: Node, binding: Mapping[str, int]):
    """Mathematical-mode evaluation with the reference's short-circuit
    and error behaviour (sym/expr.py:332-383)."""

    def go(n: Node):
        t = n[0]
        if t == "c":
            return n[1]
        if t == "s":
            try:
                return binding[n[1]]
            except KeyError:
                raise EvalError(f"no binding for symbol {n[1]}") from None
        if t == "b":
            return apply_binop(n[1], go(n[2]), go(n[3]))
        if t == "x":
            v = go(n[1])
            w = n[2]
            if is_float(w):
                return Fraction(v)
            if is_float(width_of(n[1])):
                return int(v)
            return v
        if t == "p":
            return 1 if _CMP[n[1]](go(n[2]), go(n[3])) else 0
        if t == "o":
            if n[1] == "not":
                return 0 if go(n[2][0]) else 1
            if n[1] == "and":
                for a in n[2]:
                    if not go(a):
                        return 0
                return 1
            for a in n[2]:
                if go(a):
                    return 1
            return 0
        if t == "i":
            return go(n[2]) if go(n[1]) else go(n[3])
        raise TypeError(f"not an IR node: {n!r}")

    return go(e)


def is_model(assertions: Sequence[Node], model: Mapping[str, int]) -> bool:
    """The per-instance predicate: every symbol inside its width and every
    assertion truthy, any EvalError making it false (solver/query.py:45-62)."""
    syms: Dict[str, str] = {}
    for a in assertions:
        symbols_of(a, syms)
    for name, w in syms.items():
        if is_float(w) or name not in model:
            continue
        lo, hi = bounds(w)
        if not lo <= model[name] <= hi:
            return False
    try:
        return all(evaluate(a, model) for a in assertions)
    except EvalError:
        return False


# -- simplification (restates sym/expr.py:443-585 so component splits match) -----------

def _fits(v, w: str) -> bool:
    if is_float(w):
        return True
    if not isinstance(v, int):
        return False
    lo, hi = bounds(w)
    return lo <= v <= hi


def _const_binop(e: Node, a: Node, b: Node) -> Optional[Node]:
    """sym/expr.py:452-469"""
    op, w = e[1], e[4]
    if is_float(w):
        if op in ("mod", "emod", "shl", "shr"):
            return None
        if op == "div" and b[1] == 0:
            return None
        return ("c", Fraction(apply_binop(op, a[1], b[1])), w)
    if op in _WRAP_HOM_OPS:
        return ("c", apply_binop(op, a[1], b[1]), w)
    if not (_fits(a[1], a[2]) and _fits(b[1], b[2])):
        return None
    try:
        r = apply_binop(op, a[1], b[1])
    except EvalError:
        return None
    return ("c", r, w)


def _zero(w: str):
    return Fraction(0) if is_float(w) else 0


def _simplify_node(e: Node) -> Node:
    """One-level rewrite, children already simplified (sym/expr.py:472-575)."""
    t = e[0]
    if t == "b":
        op, a, b, w = e[1], e[2], e[3], e[4]
        ca = a if a[0] == "c" else None
        cb = b if b[0] == "c" else None
        if ca is not None and cb is not None:
            folded = _const_binop(e, ca, cb)
            if folded is not None:
                return folded
        if op == "add":
            if ca is not None and ca[1] == 0:
                return b
            if cb is not None and cb[1] == 0:
                return a
            if cb is not None and a[0] == "b" and a[1] == "add" \
                    and a[3][0] == "c" and a[4] == w:
                return ("b", "add", a[2], ("c", a[3][1] + cb[1], w), w)
        elif op == "sub":
            if cb is not None and cb[1] == 0:
                return a
            if a == b and not is_float(w):
                return ("c", 0, w)
        elif op == "mul":
            if ca is not None:
                if ca[1] == 1:
                    return b
                if ca[1] == 0:
                    return ("c", _zero(w), w)
            if cb is not None:
                if cb[1] == 1:
                    return a
                if cb[1] == 0:
                    return ("c", _zero(w), w)
                if a[0] == "b" and a[1] == "mul" and a[3][0] == "c" and a[4] == w:
                    return ("b", "mul", a[2], ("c", a[3][1] * cb[1], w), w)
        elif op == "div":
            if cb is not None and cb[1] == 1:
                return a
        elif op in ("shl", "shr"):
            if cb is not None and cb[1] == 0:
                return a
        return e
    if t == "x":
        arg, w = e[1], e[2]
        if width_of(arg) == w:
            return arg
        if arg[0] == "c":
            v = arg[1]
            if is_float(w):
                return ("c", Fraction(v), w)
            if is_float(arg[2]):
                q = int(v)
                return ("c", q, w) if _fits(q, w) else e
            return ("c", v, w)
        return e
    if t == "p":
        l, r = e[2], e[3]
        if l[0] == "c" and r[0] == "c":
            if is_float(l[2]) or (_fits(l[1], l[2]) and _fits(r[1], r[2])):
                return ("c", 1 if _CMP[e[1]](l[1], r[1]) else 0, "bool")
        return e
    if t == "o":
        if e[1] == "not":
            (a,) = e[2]
            if a[0] == "c":
                return ("c", 0 if a[1] else 1, "bool")
            if a[0] == "o" and a[1] == "not":
                return a[2][0]
            return e
        absorb = 0 if e[1] == "and" else 1
        unit = 1 - absorb
        flat: List[Node] = []
        for a in e[2]:
            if a[0] == "c":
                if a[1] == absorb:
                    return ("c", absorb, "bool")
                continue
            if a[0] == "o" and a[1] == e[1]:
                flat.extend(a[2])
            else:
                flat.append(a)
        if not flat:
            return ("c", unit, "bool")
        if len(flat) == 1:
            return flat[0]
        return ("o", e[1], tuple(flat))
    if t == "i":
        if e[1][0] == "c":
            return e[2] if e[1][1] else e[3]
        if e[2] == e[3]:
            return e[2]
        return e
    return e


def simplify(e: Node) -> Node:
    scope = CompileScope._active
    memo: Dict[Node, Node] = scope.simplify if scope is not None else {}

    def go(n: Node) -> Node:
        got = memo.get(n)
        if got is not None:
            return got
        kids = children(n)
        m = n
        if kids:
            new = tuple(go(c) for c in kids)
            if new != kids:
                m = rebuild(n, new)
        r = _simplify_node(m)
        memo[n] = r
        return r

    return go(e)


# -- rendering (restates sym/expr.py:592-639; used for cache keys and goldens) -----------

def _render_fraction(v: Fraction) -> str:
    if v.denominator == 1:
        return f"{v.numerator}.0"
    d = v.denominator
    for p in (2, 5):
        while d % p == 0:
            d //= p
    if d != 1:
        return f"{v.numerator}/{v.denominator}"
    num, den = v.numerator, v.denominator
    ex = 0
    while num % den:
        num *= 10
        ex += 1
    num //= den
    sign = "-" if num < 0 else ""
    digits = str(abs(num)).rjust(ex + 1, "0")
    return f"{sign}{digits[:-ex]}.{digits[-ex:]}"


def render(e: Node) -> str:
    t = e[0]
    if t == "c":
        if e[2] == "bool":
            return "true" if e[1] else "false"
        if is_float(e[2]):
            return f"{_render_fraction(Fraction(e[1]))}:{e[2]}"
        if e[2] == "i32":
            return str(e[1])
        return f"{e[1]}:{e[2]}"
    if t == "s":
        return e[1]
    if t == "b":
        return f"({e[1]}.{e[4]} {render(e[2])} {render(e[3])})"
    if t == "x":
        return f"(cast.{e[2]} {render(e[1])})"
    if t == "p":
        return f"({e[1]}.{width_of(e[2])} {render(e[2])} {render(e[3])})"
    if t == "o":
        return f"({e[1]} {' '.join(render(a) for a in e[2])})"
    if t == "i":
        return f"(ite.{e[4]} {render(e[1])} {render(e[2])} {render(e[3])})"
    raise TypeError(f"not an IR node: {e!r}")


# -- JSON wire form ----------------------------------------------------------------------

def to_json(e: Node):
    t = e[0]
    if t == "c":
        v = e[1]
        if isinstance(v, Fraction):
            return ["c", {"f": f"{v.numerator}/{v.denominator}"}, e[2]]
        return ["c", v, e[2]]
    if t == "s":
        return ["s", e[1], e[2]]
    if t == "b":
        return ["b", e[1], to_json(e[2]), to_json(e[3]), e[4]]
    if t == "x":
        return ["x", to_json(e[1]), e[2]]
    if t == "p":
        return ["p", e[1], to_json(e[2]), to_json(e[3])]
    if t == "o":
        return ["o", e[1], [to_json(a) for a in e[2]]]
    if t == "i":
        return ["i", to_json(e[1]), to_json(e[2]), to_json(e[3]), e[4]]
    raise TypeError(f"not an IR node: {e!r}")


def from_json(j) -> Node:
    t = j[0]
    if t == "c":
        v = j[1]
        if isinstance(v, dict):
            n, d = v["f"].split("/")
            return ("c", Fraction(int(n), int(d)), j[2])
        if is_float(j[2]):
            return ("c", Fraction(v), j[2])
        return ("c", int(v), j[2])
    if t == "s":
        return ("s", j[1], j[2])
    if t == "b":
        return ("b", j[1], from_json(j[2]), from_json(j[3]), j[4])
    if t == "x":
        return ("x", from_json(j[1]), j[2])
    if t == "p":
        return ("p", j[1], from_json(j[2]), from_json(j[3]))
    if t == "o":
        return ("o", j[1], tuple(from_json(a) for a in j[2]))
    if t == "i":
        return ("i", from_json(j[1]), from_json(j[2]), from_json(j[3]), j[4])
    raise ValueError(f"bad IR json: {j!r}")


# -- conversion from the reference's expression objects ---------------------------------

def from_ref(e) -> Node:
    """Convert a ``minikernel.sym.expr`` tree (duck-typed by class name, so
    this module never imports the reference)."""
    memo: Dict[int, Node] = {}

    def go(n) -> Node:
        key = id(n)
        got = memo.get(key)
        if got is not None:
            return got
        cls = type(n).__name__
        if cls == "Const":
            r = ("c", n.value, n.width.name)
        elif cls == "Sym":
            r = ("s", n.name, n.width.name)
        elif cls == "BinOp":
            r = ("b", n.op, go(n.lhs), go(n.rhs), n.width.name)
        elif cls == "Cast":
            r = ("x", go(n.arg), n.width.name)
        elif cls == "Cmp":
            r = ("p", n.op, go(n.lhs), go(n.rhs))
        elif cls == "BoolOp":
            r = ("o", n.op, tuple(go(a) for a in n.args))
        elif cls == "Ite":
            r = ("i", go(n.cond), go(n.then), go(n.other), n.width.name)
        else:
            raise TypeError(f"not a reference expression: {n!r}")
        memo[key] = r
        return r

    return go(e)
