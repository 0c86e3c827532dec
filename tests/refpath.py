"""Locate the reference MiniKernel front end for end-to-end tests: the
offline install under baseline/_ref (travels to the GPU box) or, in the
build container only, the read-only checkout.

A workload directory holds ``kernel.mk`` + ``ctx.json``, or a
``variant.json`` naming a base workload and a front-end perturbation that
both arms (the reference and the B200 drop-in) run under:

  screen = "sat_as_unknown"   every satisfiable branch / loop screen
                              (engine/executor.py:489-492) is reported as
                              ``unknown``; the executor explores exactly the
                              same branches but sets ``state.unknown_path``
                              (engine/executor.py:588-619, :655-750), so sat
                              findings take ``_proven``'s unknown-with-witness
                              rule (engine/detectors.py:59-65)."""
import contextlib
import json
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


def workload_sources(name):
    """(kernel source, context JSON text, variant dict or None)."""
    wdir = os.path.join(ROOT, "workloads", name)
    variant = None
    vpath = os.path.join(wdir, "variant.json")
    if os.path.exists(vpath):
        variant = json.load(open(vpath))
        wdir = os.path.join(ROOT, "workloads", variant["base"])
    return (open(os.path.join(wdir, "kernel.mk")).read(),
            open(os.path.join(wdir, "ctx.json")).read(), variant)


@contextlib.contextmanager
def front_end_variant(variant):
    """Apply a variant's front-end perturbation around whatever screening is
    installed (the reference's, or GpuDetectors' with screening=True)."""
    if not variant or variant.get("screen") != "sat_as_unknown":
        yield
        return
    import minikernel.engine.executor as X

    inner = X.Executor._screen

    def _screen(self, state, cond):
        got = inner(self, state, cond)
        return "unknown" if got == "sat" else got

    X.Executor._screen = _screen
    try:
        yield
    finally:
        X.Executor._screen = inner


def analyze_workload(name, budget_s=3600.0):
    from minikernel.context import context_from_json
    from minikernel.engine import Budget, analyze
    from minikernel.lang import parse_unit, typecheck

    src, ctx_text, variant = workload_sources(name)
    unit = typecheck(parse_unit(src, "kernel.mk"))
    ctx = context_from_json(ctx_text)
    with front_end_variant(variant):
        rep = analyze(unit, ctx=ctx, budget=Budget(wall_s=budget_s))
    return json.loads(rep.to_json())
