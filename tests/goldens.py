"""Shared access to the reference goldens (tests/golden/*.json)."""
import json
import os

from paper_2603_24595_b200 import ir
from paper_2603_24595_b200.order import origin_lookup

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


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


def mismatches(doc, results):
    bad = []
    for i, (s, r) in enumerate(zip(doc["sites"], results)):
        if r.status != s["verdict"]:
            bad.append((i, s["line"], s["col"], s["verdict"], r.status))
        elif r.status == "sat" and r.witness != s.get("witness"):
            bad.append((i, s["line"], s["col"], s.get("witness"), r.witness))
    return bad
