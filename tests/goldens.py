"""Shared access to the reference goldens (tests/golden/*.json).

Parity is bit-exact against the reference's verdict and canonical witness
for every site the reference decided.  A site the reference could not
decide within its own wall budget (``reason == "solver timeout"``,
solver/interface.py:23, engine/detectors.py:126-130) is pinned instead by
the reference's external-SMT path with z3 (oracle/z3_crosscheck.py records
``z3_verdict``): the B200 stage must return that verdict."""
import json
import os

from paper_2603_24595_b200 import ir
from paper_2603_24595_b200.order import origin_lookup

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SITE_KIND = {"arithmetic_site": "IntegerOverflow", "narrowing_site": "IntegerOverflow",
             "access_site": "OutOfBounds", "store_site": "DataRace",
             "deref_site": "InvalidDeref"}


def workloads():
    """Golden workloads recorded from the reference front end (kernel.mk +
    ctx.json under workloads/); random_small.json has its own format."""
    return sorted(f[:-5] for f in os.listdir(GOLDEN)
                  if f.endswith(".json") and not f.startswith("random"))


def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


def queries(doc):
    return [([ir.from_json(a) for a in s["query"]], origin_lookup(s["origins"]))
            for s in doc["sites"]]


def timed_out(s):
    return s["verdict"] == "unknown" and s.get("reason") == "solver timeout" \
        and s.get("z3_verdict") in ("sat", "unsat")


def expected(s):
    """(verdict, witness) the B200 stage must return for a recorded site."""
    if timed_out(s):
        return s["z3_verdict"], None
    return s["verdict"], s.get("witness")


def mismatches(doc, results):
    bad = []
    for i, (s, r) in enumerate(zip(doc["sites"], results)):
        verdict, witness = expected(s)
        if r.status != verdict:
            bad.append((i, s["line"], s["col"], verdict, r.status))
        elif r.status == "sat" and witness is not None and r.witness != witness:
            bad.append((i, s["line"], s["col"], witness, r.witness))
        elif r.status == "sat" and witness is None and not ir.is_model(
                [ir.from_json(a) for a in s["query"]], r.witness):
            bad.append((i, s["line"], s["col"], "model", r.witness))
    return bad


def expected_findings(doc):
    """The reference's findings; where the reference timed out on a query
    that z3 decides, the findings of the reference's own analyze() with those
    queries answered (``findings_pinned``, oracle/z3_crosscheck.py)."""
    if "findings_pinned" in doc:
        return doc["findings_pinned"]
    return _expected_findings_dropped(doc)


def _expected_findings_dropped(doc):
    """The reference's findings, minus the ``unknown`` findings of sites the
    reference only timed out on and z3 proves unsat."""
    decided_unsat, live = set(), set()
    for s in doc["sites"]:
        key = (SITE_KIND[s["site"]], s["line"], s["col"])
        if timed_out(s) and s["z3_verdict"] == "unsat":
            decided_unsat.add(key)
        elif expected(s)[0] != "unsat":
            live.add(key)
    drop = decided_unsat - live
    return [f for f in doc["findings"]
            if not (f["status"] == "unknown" and (f["kind"], f["line"], f["column"]) in drop)]
