"""Fingerprint of the site compiler's output (light and full) on every golden
workload: compiler refactors must leave it unchanged.  Prints one JSON object
workload -> sha256 over every site's compiled query (group statuses, problem
boxes, bytecode, rows)."""
import hashlib
import json
import os
import sys
from multiprocessing import Pool

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _digest(name):
    from goldens import load, queries
    from paper_2603_24595_b200.engine import _compile_one

    h = hashlib.sha256()
    for a, o in queries(load(name)):
        for light in (True, False):
            cq, err = _compile_one((a, o, light))
            if cq is None:
                h.update(repr(("none", err)).encode())
                continue
            h.update(repr([(g.status, g.reason, g.problems, [(x[0], sorted(x[1]), x[2]) for x in g.alts])
                           for g in cq.groups]).encode())
            for p in cq.problems:
                h.update(repr((p.var_names, p.lo, p.hi, p.maximize, p.insns, p.consts, p.nregs,
                               p.atom_regs, p.atom_masks, p.rows, p.narrow, p.any_model)).encode())
            h.update(repr((cq.witness_names, cq.order, sorted(cq.defs.items()),
                           sorted(cq.free_default.items()))).encode())
    return name, h.hexdigest()[:16]


if __name__ == "__main__":
    from goldens import workloads

    names = sys.argv[1:] or workloads()
    with Pool(min(16, os.cpu_count() or 1)) as pool:
        print(json.dumps(dict(sorted(pool.map(_digest, names))), indent=0))
