"""The C oracle (oracle/mk_oracle.c) is pinned against the reference's own
verdicts and canonical witnesses on seeded random small queries
(tests/golden/random_small.json, made by oracle/gen_random.py), and the
compiler + search logic (host emulation) is checked against both."""
import os

import pytest

from goldens import GOLDEN
from refpath import ROOT

import json

EMU = os.path.join(ROOT, "tests", "emu", "libmk_emu.so")


def _fixtures():
    with open(os.path.join(GOLDEN, "random_small.json")) as fh:
        return json.load(fh)["queries"]


def _oracle(q):
    from oracle import c_oracle
    from paper_2603_24595_b200 import ir
    from paper_2603_24595_b200.order import optimization_order, origin_lookup

    assertions = [ir.from_json(a) for a in q["query"]]
    widths = {}
    for a in assertions:
        ir.symbols_of(a, widths)
    order = optimization_order(widths, origin_lookup(q["origins"]))
    box = {k: tuple(v) for k, v in q["box"].items()}
    return c_oracle.lexmin([ir.render(a) for a in assertions], order, box)


def test_oracle_pinned_to_reference():
    bad = []
    qs = _fixtures()
    assert len(qs) >= 200
    for i, q in enumerate(qs):
        got = _oracle(q)
        assert got is not None, i
        status, witness, _ = got
        if status != q["verdict"] or (status == "sat" and witness != q["witness"]):
            bad.append((i, status, q["verdict"]))
    assert bad == []


def test_emulated_engine_matches_random_fixtures():
    from paper_2603_24595_b200 import ir
    from paper_2603_24595_b200.engine import SiteChecker
    from paper_2603_24595_b200.order import origin_lookup

    chk = SiteChecker(lib_path=EMU)
    qs = _fixtures()
    res = chk.check_queries([([ir.from_json(a) for a in q["query"]], origin_lookup(q["origins"]))
                             for q in qs])
    bad = [(i, r.status, q["verdict"]) for i, (q, r) in enumerate(zip(qs, res))
           if r.status != q["verdict"] or (r.status == "sat" and r.witness != q["witness"])]
    assert bad == []


@pytest.mark.gpu
def test_gpu_engine_matches_random_fixtures():
    from paper_2603_24595_b200 import ir
    from paper_2603_24595_b200.engine import SiteChecker
    from paper_2603_24595_b200.order import origin_lookup

    chk = SiteChecker(device=0)
    qs = _fixtures()
    try:
        res = chk.check_queries([([ir.from_json(a) for a in q["query"]],
                                  origin_lookup(q["origins"])) for q in qs])
    finally:
        chk.close()
    bad = [(i, r.status, q["verdict"]) for i, (q, r) in enumerate(zip(qs, res))
           if r.status != q["verdict"] or (r.status == "sat" and r.witness != q["witness"])]
    assert bad == []
