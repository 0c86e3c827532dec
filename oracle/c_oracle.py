"""ctypes wrapper of the C oracle (oracle/mk_oracle.c).  TEST INFRASTRUCTURE
ONLY: the brute-force lexicographic optimum of a query over a small box."""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Callable, Dict, List, Optional, Sequence, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libmk_oracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        _lib = ctypes.CDLL(LIB)
        _lib.mko_lexmin.argtypes = [ctypes.c_char_p, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_char_p),
                                    ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                    ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64)]
    return _lib


def available() -> bool:
    try:
        _load()
        return True
    except Exception:
        return False


def _words(v: int) -> Tuple[int, int]:
    lo = v & 0xFFFFFFFFFFFFFFFF
    if lo >= 1 << 63:
        lo -= 1 << 64
    return lo, v >> 64


def lexmin(rendered: Sequence[str], order: Sequence[Tuple[str, str]],
           box: Dict[str, Tuple[int, int]], limit: int = 1 << 26):
    """(status, witness, evaluated) with status sat/unsat, or None when the
    oracle cannot decide (unsupported text, >128-bit arithmetic, box too big)."""
    lib = _load()
    n = len(order)
    names = (ctypes.c_char_p * max(n, 1))(*[o[0].encode() for o in order])
    mx = (ctypes.c_int * max(n, 1))(*[1 if o[1] == "max" else 0 for o in order])
    lo = (ctypes.c_int64 * max(2 * n, 1))()
    hi = (ctypes.c_int64 * max(2 * n, 1))()
    for i, (name, _) in enumerate(order):
        a, b = box[name]
        lo[2 * i], lo[2 * i + 1] = _words(a)
        hi[2 * i], hi[2 * i + 1] = _words(b)
    point = (ctypes.c_int64 * max(2 * n, 1))()
    ev = ctypes.c_int64(0)
    text = "\n".join(rendered).encode()
    rc = lib.mko_lexmin(text, n, names, mx, lo, hi, limit, point, ctypes.byref(ev))
    if rc < 0:
        return None
    if rc == 0:
        return "unsat", {}, ev.value
    w = {}
    for i, (name, _) in enumerate(order):
        w[name] = (int(point[2 * i + 1]) << 64) | (int(point[2 * i]) & 0xFFFFFFFFFFFFFFFF)
    return "sat", {k: w[k] for k in sorted(w)}, ev.value


def box_from_atoms(assertions, widths: Dict[str, str]) -> Dict[str, Tuple[int, int]]:
    """Every model satisfies every top-level atom, so symbol bounds stated by
    unary comparison atoms, clipped to the widths, enclose all models."""
    from paper_2603_24595_b200 import ir

    box = {n: ir.bounds(w) for n, w in widths.items() if not ir.is_float(w)}
    flip = {"lt": "gt", "le": "ge", "gt": "lt", "ge": "le", "eq": "eq"}
    todo = [ir.simplify(a) for a in assertions]
    while todo:
        a = todo.pop()
        if a[0] == "o" and a[1] == "and":
            todo.extend(a[2])
            continue
        if a[0] != "p":
            continue
        op, l, r = a[1], a[2], a[3]
        if l[0] == "c" and r[0] == "s":
            l, r, op = r, l, flip.get(op, op)
        if not (l[0] == "s" and r[0] == "c") or l[1] not in box or not isinstance(r[1], int):
            continue
        lo, hi = box[l[1]]
        v = r[1]
        if op == "eq":
            lo, hi = max(lo, v), min(hi, v)
        elif op == "le":
            hi = min(hi, v)
        elif op == "lt":
            hi = min(hi, v - 1)
        elif op == "ge":
            lo = max(lo, v)
        elif op == "gt":
            lo = max(lo, v + 1)
        box[l[1]] = (lo, hi)
    return box


def lexmin_small(assertions, origin_of: Callable[[str], str], box_limit: int = 1 << 22):
    """Oracle verdict of an IR query when its atom-derived box is small
    enough, else None."""
    from paper_2603_24595_b200 import ir
    from paper_2603_24595_b200.order import optimization_order

    widths: Dict[str, str] = {}
    for a in assertions:
        ir.symbols_of(a, widths)
    if any(ir.is_float(w) for w in widths.values()):
        return None
    order = optimization_order(widths, origin_of)
    box = box_from_atoms(assertions, widths)
    vol = 1
    for n, _ in order:
        lo, hi = box[n]
        if hi < lo:
            return "unsat", {}
        vol *= hi - lo + 1
        if vol > box_limit:
            return None
    got = lexmin([ir.render(a) for a in assertions], order, box, limit=box_limit)
    if got is None:
        return None
    return got[0], got[1]
