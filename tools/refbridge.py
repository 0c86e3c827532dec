"""Bridge to the UNMODIFIED reference checker for bench.py's reference arm
and CPU baseline: rebuilds each recorded site query as reference expression
objects and runs the reference's own decision + canonicalisation
(solver/interface.py:49 Solver.check, engine/report.py:147
canonicalize_witness), one Solver per step as in one analysis run
(engine/executor.py:114)."""
from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def have_reference() -> bool:
    for p in (REF, "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "minikernel")):
            if p not in sys.path:
                sys.path.insert(0, p)
            return True
    return False


def to_ref(e, E):
    t = e[0]
    W = E.WIDTH_BY_NAME if hasattr(E, "WIDTH_BY_NAME") else None
    if t == "c":
        return E.Const(e[1], W[e[2]])
    if t == "s":
        return E.Sym(e[1], W[e[2]])
    if t == "b":
        return E.BinOp(e[1], to_ref(e[2], E), to_ref(e[3], E), W[e[4]])
    if t == "x":
        return E.Cast(to_ref(e[1], E), W[e[2]])
    if t == "p":
        return E.Cmp(e[1], to_ref(e[2], E), to_ref(e[3], E))
    if t == "o":
        return E.BoolOp(e[1], tuple(to_ref(a, E) for a in e[2]))
    if t == "i":
        return E.Ite(to_ref(e[1], E), to_ref(e[2], E), to_ref(e[3], E), W[e[4]])
    raise ValueError(t)


def reference_check_queries(queries, budget_s=None):
    """Decide queries in order with the reference; returns (count, results)."""
    have_reference()
    from minikernel.engine.report import canonicalize_witness
    from minikernel.engine.state import SymbolTable
    from minikernel.solver.interface import Solver
    from minikernel.sym import expr as E
    from paper_2603_24595_b200 import ir

    solver = Solver()
    out = []
    t0 = time.perf_counter()
    for assertions, origin_of in queries:
        if budget_s is not None and out and time.perf_counter() - t0 > budget_s:
            break
        ref = [to_ref(a, E) for a in assertions]
        table = SymbolTable()
        names = {}
        for a in assertions:
            ir.symbols_of(a, names)
        for n in names:
            o = origin_of(n)
            if o != "unknown":
                table.origins[n.rstrip("'")] = o
        v = solver.check(ref)
        w = canonicalize_witness(solver, ref, v, table) if v.is_sat else {}
        out.append((v.status, w))
    return len(out), out
