"""Independent cross-check of reference-timeout sites.  TEST INFRASTRUCTURE ONLY.

The reference's builtin solver gives up after ``SolverOptions.timeout_s``
(30 s, solver/interface.py:23) and the site is reported ``unknown``
(engine/detectors.py:126-130, :157-162, :228-232).  Whether a query times out
depends on the host CPU, not on the query, so the B200 stage is allowed to
decide such a site.  To pin that decision to something other than our own
engine, this script hands the SAME recorded query to the reference's own
external-SMT path (solver/external.py:94-146 ExternalSolver with z3, the
SMT-LIB encoding of solver/smtlib.py:114-144) with a long timeout, and
records the verdict as ``z3_verdict`` (plus ``z3_model`` when sat) in the
golden fixture.  z3 itself is not needed on the GPU box: the verdict travels
in tests/golden/<workload>.json.

Usage:  python oracle/z3_crosscheck.py <workload> [timeout_s]
"""
from __future__ import annotations

import json
import os
import shutil
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main(argv) -> None:
    name = argv[0]
    if "--pinned-only" in argv:
        from refbridge import have_reference

        assert have_reference(), "reference MiniKernel not found"
        path = os.path.join(ROOT, "tests", "golden", f"{name}.json")
        doc = json.load(open(path))
        doc["findings_pinned"] = pinned_findings(name, doc)
        with open(path, "w") as fh:
            json.dump(doc, fh, separators=(",", ":"))
            fh.write("\n")
        print(name, "findings_pinned", doc["findings_pinned"])
        return
    timeout = float(argv[1]) if len(argv) > 1 else 900.0
    from refbridge import have_reference, to_ref

    assert have_reference(), "reference MiniKernel not found"
    from minikernel.solver.interface import Solver, SolverOptions
    from minikernel.sym import expr as E

    from paper_2603_24595_b200 import ir

    z3 = shutil.which("z3")
    assert z3, "z3 not on PATH"
    path = os.path.join(ROOT, "tests", "golden", f"{name}.json")
    doc = json.load(open(path))
    for i, s in enumerate(doc["sites"]):
        if s["verdict"] != "unknown" or s.get("reason") != "solver timeout":
            continue
        solver = Solver(SolverOptions(timeout_s=timeout, external_cmd=[z3, "-in"]))
        ref = [to_ref(ir.from_json(a), E) for a in s["query"]]
        t0 = time.monotonic()
        v = solver.check(ref)
        solver.close()
        s["z3_verdict"] = v.status
        s["z3_s"] = round(time.monotonic() - t0, 3)
        if v.is_sat and v.model:
            s["z3_model"] = {k: int(x) for k, x in v.model.items()}
        print(f"{name} site {i} line {s['line']}:{s['col']} {s['site']}: reference "
              f"{s['verdict']} ({s['reason']}), z3 {v.status} in {s['z3_s']}s", flush=True)
    doc["findings_pinned"] = pinned_findings(name, doc)
    with open(path, "w") as fh:
        json.dump(doc, fh, separators=(",", ":"))
        fh.write("\n")


def pinned_findings(name, doc):
    """The reference's own analyze() (front end, Detectors, merge_findings,
    engine/report.py:109-140) with every timed-out query answered by its z3
    verdict instead: the findings the reference reports when its solver is
    given the time it needs.  Stored as ``findings_pinned``."""
    from refbridge import to_ref
    from minikernel.solver import interface as SI
    from minikernel.solver.query import Verdict
    from minikernel.sym import expr as E

    from paper_2603_24595_b200 import ir

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from refpath import analyze_workload

    pins = {}
    for s in doc["sites"]:
        if s.get("reason") == "solver timeout" and s.get("z3_verdict") == "unsat":
            key = tuple(E.render(to_ref(ir.from_json(a), E)) for a in s["query"])
            pins[key] = Verdict.unsat()
    orig = SI.Solver.check

    z3 = shutil.which("z3")
    from minikernel.solver.interface import Solver, SolverOptions

    def check(self, assertions, bounds=None):
        got = pins.get(tuple(E.render(a) for a in assertions))
        if got is not None and not bounds:
            return got
        got = orig(self, assertions, bounds)
        # the builtin solver's 30 s timeout depends on the host's load, so a
        # query it decided in the recording run may time out here: ask z3
        # for those too (sat answers keep the reference's own path: only an
        # unsat z3 verdict replaces the unknown)
        if got.status == "unknown" and "timeout" in (getattr(got, "reason", "") or "") \
                and not bounds and z3:
            zs = Solver(SolverOptions(timeout_s=600.0, external_cmd=[z3, "-in"]))
            try:
                v = zs.check(list(assertions))
            finally:
                zs.close()
            if v.status == "unsat":
                return v
        return got

    SI.Solver.check = check
    try:
        return analyze_workload(name)["findings"]
    finally:
        SI.Solver.check = orig


if __name__ == "__main__":
    main(sys.argv[1:])
