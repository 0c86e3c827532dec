"""Seeded random small checker queries decided by the UNMODIFIED reference.
TEST INFRASTRUCTURE ONLY.

Each query mimics the shape of a checker site query (engine/detectors.py):
context counts (BS/SL/TC), scalar arguments, thread identities (some with
race twins), loop indices and havoc loads, each bounded by explicit atoms to a
small box, plus random arithmetic / comparison / boolean atoms using every
operator of the expression algebra (sym/expr.py:87-89) including truncating
div/mod, Euclidean emod and constant shifts.  The reference decides each one
with ``Solver.check`` (solver/interface.py:49) and, when satisfiable, pins
the canonical witness with ``canonicalize_witness`` (engine/report.py:147).
Undecided (``unknown``) queries are dropped.

Writes tests/golden/random_small.json.  Usage: python oracle/gen_random.py [N] [seed]
"""

from __future__ import annotations

import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

POOL = [
    # name, width, origin, (lo, hi) box
    ("BS", "i64", "context", (1, 3)),
    ("SL", "i64", "context", (1, 6)),
    ("n", "i32", "scalar-arg", (-3, 9)),
    ("m", "i32", "scalar-arg", (0, 5)),
    ("blockIdx.x", "i32", "thread-id", (0, 4)),
    ("threadIdx.x", "i32", "thread-id", (0, 7)),
    ("threadIdx.y", "i32", "thread-id", (0, 2)),
    ("i$1", "i32", "loop-index", (-2, 6)),
    ("ld$2", "i32", "havoc", (-4, 4)),
    ("t.numel", "i64", "tensor-field", (1, 8)),
]
TWINS = {"blockIdx.x", "threadIdx.x", "threadIdx.y", "i$1", "ld$2"}


def _to_ref(e, E):
    t = e[0]
    W = {"i32": E.I32, "i64": E.I64, "bool": E.BOOL}
    if t == "c":
        return E.Const(e[1], W[e[2]])
    if t == "s":
        return E.Sym(e[1], W[e[2]])
    if t == "b":
        return E.BinOp(e[1], _to_ref(e[2], E), _to_ref(e[3], E), W[e[4]])
    if t == "x":
        return E.Cast(_to_ref(e[1], E), W[e[2]])
    if t == "p":
        return E.Cmp(e[1], _to_ref(e[2], E), _to_ref(e[3], E))
    if t == "o":
        return E.BoolOp(e[1], tuple(_to_ref(a, E) for a in e[2]))
    raise ValueError(t)


def _rand_expr(rng, syms, depth):
    if depth <= 0 or rng.random() < 0.3:
        if rng.random() < 0.65:
            n, w = rng.choice(syms)
            return ("s", n, w)
        return ("c", rng.randint(-6, 9), "i64" if rng.random() < 0.3 else "i32")
    op = rng.choice(["add", "add", "sub", "mul", "mul", "div", "mod", "emod", "shl", "shr"])
    a = _rand_expr(rng, syms, depth - 1)
    if op in ("shl", "shr"):
        b = ("c", rng.randint(0, 3), "i32")
    elif op in ("div", "mod", "emod") and rng.random() < 0.6:
        b = ("c", rng.choice([-3, -2, 2, 3, 4, 5, 8]), "i32")
    else:
        b = _rand_expr(rng, syms, depth - 1)
    w = "i64" if rng.random() < 0.3 else "i32"
    e = ("b", op, a, b, w)
    if rng.random() < 0.15:
        e = ("x", e, "i64" if w == "i32" else "i32")
    return e


def _rand_atom(rng, syms, depth):
    r = rng.random()
    if r < 0.15:
        return ("o", "or", (_rand_atom(rng, syms, depth - 1), _rand_atom(rng, syms, depth - 1)))
    if r < 0.22:
        return ("o", "not", (("o", "and", (_rand_atom(rng, syms, depth - 1),
                                           _rand_atom(rng, syms, depth - 1))),))
    op = rng.choice(["eq", "ne", "lt", "le", "gt", "ge"])
    return ("p", op, _rand_expr(rng, syms, depth), _rand_expr(rng, syms, depth))


def make_query(rng):
    k = rng.randint(2, 6)
    chosen = rng.sample(POOL, k)
    twin = rng.random() < 0.25
    syms, origins, atoms, box = [], {}, [], {}
    for name, w, origin, (lo, hi) in chosen:
        syms.append((name, w))
        origins[name] = origin
        box[name] = (lo, hi)
        if twin and name in TWINS:
            syms.append((name + "'", w))
            box[name + "'"] = (lo, hi)
    for name, w in syms:
        lo, hi = box[name]
        atoms.append(("p", "ge", ("s", name, w), ("c", lo, w)))
        atoms.append(("p", "le", ("s", name, w), ("c", hi, w)))
    if "BS" in origins and "SL" in origins and rng.random() < 0.5:
        # the context law TC = BS*SL (context.py:523)
        syms.append(("TC", "i64"))
        origins["TC"] = "context"
        box["TC"] = (1, 18)
        atoms.append(("p", "eq", ("s", "TC", "i64"),
                      ("b", "mul", ("s", "BS", "i64"), ("s", "SL", "i64"), "i64")))
    for _ in range(rng.randint(1, 4)):
        atoms.append(_rand_atom(rng, syms, rng.randint(1, 3)))
    if twin:
        primed = [n for n, _ in syms if n.endswith("'")]
        if primed:
            eqs = [("p", "eq", ("s", p[:-1], "i32" if p[:-1] != "t.numel" else "i64"),
                    ("s", p, "i32")) for p in primed]
            atoms.append(("o", "not", (("o", "and", tuple(eqs)) if len(eqs) > 1 else eqs[0],)))
    return atoms, origins, box


def main(argv):
    n = int(argv[0]) if argv else 300
    seed = int(argv[1]) if len(argv) > 1 else 0
    for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "minikernel")):
            sys.path.insert(0, p)
            break
    from minikernel.engine.report import canonicalize_witness
    from minikernel.engine.state import SymbolTable
    from minikernel.solver.interface import Solver
    from minikernel.sym import expr as E

    from paper_2603_24595_b200 import ir

    rng = random.Random(seed)
    out = []
    tries = 0
    t0 = time.time()
    while len(out) < n and tries < 20 * n:
        tries += 1
        atoms, origins, box = make_query(rng)
        vol = 1
        for lo, hi in box.values():
            vol *= hi - lo + 1
        if vol > (1 << 22):  # keep every fixture brute-forceable by the oracle
            continue
        try:
            ref_atoms = [_to_ref(a, E) for a in atoms]
        except Exception:
            continue
        table = SymbolTable()
        for name, origin in origins.items():
            table.origins[name] = origin
        solver = Solver()
        v = solver.check(ref_atoms)
        if v.is_unknown:
            continue
        wit = canonicalize_witness(solver, ref_atoms, v, table) if v.is_sat else {}
        full_order_box = {}
        for a in atoms:
            for s in ir.symbols_of(a):
                full_order_box[s] = box.get(s, box.get(s.rstrip("'")))
        out.append({
            "query": [ir.to_json(ir.from_ref(a)) for a in ref_atoms],
            "origins": {s: table.origin_of(s) for s in full_order_box},
            "box": {k: list(v2) for k, v2 in full_order_box.items()},
            "verdict": v.status,
            "witness": {k: int(x) for k, x in wit.items()},
        })
    path = os.path.join(ROOT, "tests", "golden", "random_small.json")
    with open(path, "w") as fh:
        json.dump({"generator": "oracle/gen_random.py", "seed": seed, "queries": out}, fh,
                  separators=(",", ":"))
        fh.write("\n")
    sat = sum(1 for q in out if q["verdict"] == "sat")
    print(f"{len(out)} queries ({sat} sat) from {tries} draws in {time.time() - t0:.1f}s -> {path}")


if __name__ == "__main__":
    main(sys.argv[1:])
