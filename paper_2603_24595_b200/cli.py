"""Command line of the B200 checking stage (the
reference specifies its CLI in SPEC.md:633-687 but does not ship it).

    python -m paper_2603_24595_b200 analyze --kernel K.mk [--wrapper W] [--context C.json]
        [--budget S] [--format json|text] [--out R.json] [--device N] [--no-screening]
    python -m paper_2603_24595_b200 infer --log RUNS.jsonl --kernel NAME --out C.json
    python -m paper_2603_24595_b200 races --kernel K.mk [--wrapper W] [--context C.json]
        --launch BS=1,SL=32[,name=value...] [--device N]
    python -m paper_2603_24595_b200 replay --kernel K.mk [--wrapper W] [--context C.json]
    python -m paper_2603_24595_b200 corpus DIR [DIR ...] [--device N]

``analyze`` runs the reference front end (parser, typechecker, executor DFS:
engine/executor.py:778-800, unchanged) with the checking stage and branch
screening on the B200 engine (``GpuDetectors``) and prints the reference's
ReportSet (engine/report.py:67-106).  Exit codes follow SPEC.md:645-646:
0 no findings, 1 findings, 2 operational error.

``infer`` is the reference's own context inference (context.py:73-110,
:315-395, :217-231) -- host arithmetic with no device value, exposed here so
the CLI covers the specified commands.

``races`` records every executed access during the analysis and replays
them at one concrete launch with the specification's oracle rule
(paper_2603_24595_b200.replay, non-parity): exit 1 when a read-write or
write-write race exists.  ``--launch`` pins launch-level symbols (BS, SL,
scalar arguments...); the rest of the launch is the canonical model of the
context's constraints.

``replay`` analyzes and then replays every sat overflow / out-of-bounds /
deref witness (paper_2603_24595_b200.witness): expression
level and over every thread of the witness's launch; exit 1 when one is not
confirmed.

``corpus`` analyzes several workload directories (kernel.mk + ctx.json each,
BASELINE.json configs[4]) on one device context, one JSON line per entry.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from typing import Dict, List, Optional


def _reference():
    try:
        import minikernel  # noqa: F401
    except ImportError:
        import os

        here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.join(here, "baseline", "_ref"))
        import minikernel  # noqa: F401


def _load(kernel: str, context: Optional[str]):
    _reference()
    from minikernel.context import context_from_json
    from minikernel.lang import parse_unit, typecheck

    with open(kernel) as fh:
        unit = typecheck(parse_unit(fh.read(), kernel))
    ctx = None
    if context:
        with open(context) as fh:
            ctx = context_from_json(fh.read(), context)
    return unit, ctx


def _analyze(unit, wrapper, ctx, budget, device, screening, recorders=None, created=None,
             record_queries=False):
    from minikernel.engine import Budget, analyze

    from .detectors import install, shared_checker, uninstall

    chk = shared_checker(device)
    prev = install(device=device, checker=chk, screening=screening, recorders=recorders,
                   created=created, record_queries=record_queries)
    try:
        b = Budget(wall_s=budget) if budget else None
        return analyze(unit, wrapper, ctx=ctx, budget=b)
    finally:
        uninstall(prev)


def cmd_analyze(a) -> int:
    unit, ctx = _load(a.kernel, a.context)
    t0 = time.perf_counter()
    rep = _analyze(unit, a.wrapper, ctx, a.budget, a.device, not a.no_screening)
    dt = time.perf_counter() - t0
    text = rep.to_json() if a.format == "json" else rep.to_text()
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    else:
        print(text)
    print(f"# {len(rep.findings)} finding(s) in {dt:.2f} s (B200 checking stage)", file=sys.stderr)
    return 1 if rep.findings else 0


def cmd_infer(a) -> int:
    _reference()
    from .context import infer_context_json

    with open(a.log) as fh:
        text = infer_context_json(fh.read(), a.kernel, a.log)
    with open(a.out, "w") as fh:
        fh.write(text)
    return 0


def _pins(spec: str) -> Dict[str, int]:
    out = {}
    for part in filter(None, (p.strip() for p in spec.split(","))):
        k, v = part.split("=", 1)
        out[k.strip()] = int(v)
    return out


def cmd_races(a) -> int:
    from . import replay
    from .detectors import shared_checker

    unit, ctx = _load(a.kernel, a.context)
    recs: List[object] = []
    _analyze(unit, a.wrapper, ctx, a.budget, a.device, True, recorders=recs)
    records = [r for d in recs for r in d.accesses]
    if not records:
        print(json.dumps({"has_race": False, "accesses": 0}))
        return 0
    origin_of = recs[0].table.origin_of
    chk = shared_checker(a.device)
    launch = replay.launch_model(chk, records, origin_of, _pins(a.launch))
    res = replay.replay_races(chk.engine, records, origin_of, launch)
    print(json.dumps({"has_race": res.has_race, "racy_granules": res.racy,
                      "accesses": res.accesses, "instances": res.instances,
                      "tuples": res.tuples, "skipped": [(r.line, r.kind, why) for r, why in res.skipped],
                      "launch": {k: v for k, v in launch.items() if "Dim" in k or k in ("BS", "SL", "TC")},
                      "first": res.first}))
    return 1 if res.has_race else 0


def cmd_replay(a) -> int:
    """SPEC.md:664 replay: analyze, then replay every sat overflow /
    out-of-bounds / deref witness (paper_2603_24595_b200.witness): expression
    level and every thread of the witness launch on the device.  Exit 1 when
    a witness is not confirmed."""
    from .detectors import shared_checker
    from .witness import replay_witness

    unit, ctx = _load(a.kernel, a.context)
    made: List[object] = []
    rep = _analyze(unit, a.wrapper, ctx, a.budget, a.device, True, created=made,
                   record_queries=True)
    chk = shared_checker(a.device)
    bad = 0
    for f in rep.findings:
        if f.status != "sat" or f.kind == "DataRace" or not f.witness:
            continue
        det = next((d for d in made if (f.kind, f.line, f.column) in d.sat_queries), None)
        if det is None:
            continue
        q = det.sat_queries[(f.kind, f.line, f.column)]
        r = replay_witness(chk.engine, q, det.table.origin_of, f.witness)
        bad += r.status == "not-confirmed"
        print(json.dumps({"kind": f.kind, "line": f.line, "column": f.column, "status": r.status,
                          "violating_threads": r.violating_threads, "candidate_threads": r.candidates,
                          "note": r.note}))
    return 1 if bad else 0


def cmd_corpus(a) -> int:
    import os

    any_findings = False
    for d in a.dirs:
        unit, ctx = _load(os.path.join(d, "kernel.mk"), os.path.join(d, "ctx.json"))
        t0 = time.perf_counter()
        rep = _analyze(unit, None, ctx, a.budget, a.device, True)
        doc = json.loads(rep.to_json())
        print(json.dumps({"entry": d, "seconds": time.perf_counter() - t0,
                          "coverage": doc.get("coverage"), "findings": doc["findings"]}))
        any_findings |= bool(doc["findings"])
    return 1 if any_findings else 0


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2603_24595_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("analyze")
    p.add_argument("--kernel", required=True)
    p.add_argument("--wrapper")
    p.add_argument("--context")
    p.add_argument("--budget", type=float)
    p.add_argument("--format", choices=["json", "text"], default="json")
    p.add_argument("--out")
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--no-screening", action="store_true")
    p = sub.add_parser("infer")
    p.add_argument("--log", required=True)
    p.add_argument("--kernel", required=True)
    p.add_argument("--out", required=True)
    p = sub.add_parser("races")
    p.add_argument("--kernel", required=True)
    p.add_argument("--wrapper")
    p.add_argument("--context")
    p.add_argument("--budget", type=float)
    p.add_argument("--launch", default="")
    p.add_argument("--device", type=int, default=0)
    p = sub.add_parser("replay")
    p.add_argument("--kernel", required=True)
    p.add_argument("--wrapper")
    p.add_argument("--context")
    p.add_argument("--budget", type=float)
    p.add_argument("--device", type=int, default=0)
    p = sub.add_parser("corpus")
    p.add_argument("dirs", nargs="+")
    p.add_argument("--budget", type=float)
    p.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        return {"analyze": cmd_analyze, "infer": cmd_infer, "races": cmd_races,
                "replay": cmd_replay, "corpus": cmd_corpus}[a.cmd](a)
    except SystemExit:
        raise
    except Exception as exc:  # operational error
        print(f"error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
