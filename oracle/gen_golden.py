"""Golden-fixture generator.  TEST INFRASTRUCTURE ONLY.

Runs the UNMODIFIED reference MiniKernel checker (``/root/reference`` or an
install of it under ``baseline/_ref``) on every workload under
``workloads/<name>/`` (``kernel.mk`` + ``ctx.json``) and records, for each
checker site call, the exact query the reference hands its solver together
with the reference's verdict and canonical witness:

    engine/detectors.py:111-125   IntegerOverflow query + witness
    engine/detectors.py:143-156   OutOfBounds query + witness
    engine/detectors.py:213-227   DataRace query + witness
    engine/detectors.py:284-293   InvalidDeref query + witness

Queries are stored in this package's JSON IR (``paper_2603_24595_b200.ir``)
together with the origin of every symbol (needed for the witness order,
engine/report.py:177-203), so the GPU parity tests need neither the
reference nor its front end at run time.  The final ``ReportSet`` findings
are stored too (the end-to-end parity artefact).

Usage:  python oracle/gen_golden.py [workload ...]
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)


def _reference_path() -> str:
    for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "minikernel")):
            return p
    raise SystemExit("reference MiniKernel not found")


def record(name: str, budget_s: float = 3600.0) -> dict:
    sys.path.insert(0, _reference_path())
    from minikernel.context import context_from_json
    from minikernel.engine import Budget, analyze
    import minikernel.engine.detectors as D
    import minikernel.solver.interface as SI
    from minikernel.lang import parse_unit, typecheck

    from paper_2603_24595_b200 import ir

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from refpath import front_end_variant, workload_sources

    src, ctx_text, variant = workload_sources(name)
    unit = typecheck(parse_unit(src, "kernel.mk"))
    ctx = context_from_json(ctx_text)

    current = [None]
    sites = []
    orig_check = SI.Solver.check
    orig_canon = D.canonicalize_witness

    def check(self, assertions, bounds=None):
        v = orig_check(self, assertions, bounds)
        cur = current[0]
        if cur is not None and "query" not in cur:
            cur["query"] = [ir.to_json(ir.from_ref(a)) for a in assertions]
            cur["verdict"] = v.status
            cur["reason"] = v.reason
        return v

    def canon(solver, assertions, base, table):
        t0 = time.monotonic()
        w = orig_canon(solver, assertions, base, table)
        cur = current[0]
        if cur is not None:
            cur["witness"] = {k: int(v) for k, v in w.items()}
            cur["canon_s"] = time.monotonic() - t0
            names = set()
            for a in assertions:
                names |= set(ir.symbols_of(ir.from_ref(a)))
            cur["origins"] = {n: table.origin_of(n) for n in sorted(names)}
        return w

    SI.Solver.check = check
    D.canonicalize_witness = canon
    wrapped = {}
    for meth in ("arithmetic_site", "narrowing_site", "access_site",
                 "store_site", "deref_site"):
        f = getattr(D.Detectors, meth)
        wrapped[meth] = f

        def wrap(self, state, *args, _f=f, _m=meth, **kw):
            line, col, text = args[-3], args[-2], args[-1]
            rec = {"site": _m, "line": line, "col": col, "text": text,
                   "unknown_path": bool(state.unknown_path)}
            current[0] = rec
            t0 = time.monotonic()
            try:
                return _f(self, state, *args, **kw)
            finally:
                rec["site_s"] = time.monotonic() - t0
                current[0] = None
                if "query" in rec:
                    if "origins" not in rec:
                        names = set()
                        for a in rec["query"]:
                            names |= set(ir.symbols_of(ir.from_json(a)))
                        rec["origins"] = {n: self.table.origin_of(n) for n in sorted(names)}
                    sites.append(rec)
        setattr(D.Detectors, meth, wrap)
    try:
        t0 = time.monotonic()
        with front_end_variant(variant):
            rep = analyze(unit, ctx=ctx, budget=Budget(wall_s=budget_s))
        wall = time.monotonic() - t0
    finally:
        SI.Solver.check = orig_check
        D.canonicalize_witness = orig_canon
        for meth, f in wrapped.items():
            setattr(D.Detectors, meth, f)
    doc = json.loads(rep.to_json())
    return {
        "workload": name,
        "generator": "oracle/gen_golden.py (reference MiniKernel, builtin solver)",
        "reference_wall_s": round(wall, 3),
        "coverage": doc["coverage"],
        "states": doc["states"] if "states" in doc else doc["budget"]["states"],
        "queries": doc["budget"]["queries"],
        "findings": doc["findings"],
        "sites": sites,
    }


def main(argv) -> None:
    names = argv or sorted(os.listdir(os.path.join(ROOT, "workloads")))
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    for name in names:
        t0 = time.time()
        doc = record(name)
        out = os.path.join(ROOT, "tests", "golden", f"{name}.json")
        with open(out, "w") as fh:
            json.dump(doc, fh, separators=(",", ":"))
            fh.write("\n")
        print(f"{name}: {len(doc['sites'])} sites, {len(doc['findings'])} findings, "
              f"coverage {doc['coverage']}, {time.time() - t0:.1f}s -> {out}")


if __name__ == "__main__":
    main(sys.argv[1:])
