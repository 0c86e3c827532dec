"""Locate the reference MiniKernel front end for end-to-end tests: the
offline install under baseline/_ref (travels to the GPU box) or, in the
build container only, the read-only checkout."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def add_reference() -> bool:
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "minikernel")):
            if p not in sys.path:
                sys.path.insert(0, p)
            return True
    return False


def analyze_workload(name, budget_s=3600.0):
    from minikernel.context import context_from_json
    from minikernel.engine import Budget, analyze
    from minikernel.lang import parse_unit, typecheck
    import json

    wdir = os.path.join(ROOT, "workloads", name)
    unit = typecheck(parse_unit(open(os.path.join(wdir, "kernel.mk")).read(), "kernel.mk"))
    ctx = context_from_json(open(os.path.join(wdir, "ctx.json")).read())
    rep = analyze(unit, ctx=ctx, budget=Budget(wall_s=budget_s))
    return json.loads(rep.to_json())
