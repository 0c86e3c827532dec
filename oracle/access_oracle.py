"""TEST INFRASTRUCTURE ONLY (never imported by the package): pure-Python
restatement of the specification's concrete-oracle race rule
(module ``oracle`` of the reference specification, which
the reference does not ship): after executing every thread of a launch,
"pair accesses in the same region at overlapping bytes from different
threads with >= 1 write, same barrier-epoch for shared memory, any epoch
for global".

Input: the access programs ``paper_2603_24595_b200.replay.build`` makes for
recorded accesses at one launch (each one thread's path + byte offset over
its private symbols).  Every instance is evaluated with the reference's
mathematical-mode semantics (package IR evaluate = sym/expr.py:332-383);
each executed access contributes its bytes [offset, offset + width).

Output: (has_race, racy granules, first race) where the granule count and
the first race follow the device's reporting conventions so tests can
compare exactly: granules of a region are ``granule`` bytes (all accesses
cover whole granules when offsets are aligned), the first race is at the
least (region, epoch, block, granule) and its pair is (the first write of
that granule in access-then-instance order, the first access of another
thread after it in the order writes-before-reads)."""

from __future__ import annotations

from typing import Dict, List, Tuple

from paper_2603_24595_b200 import ir
from paper_2603_24595_b200.race import ID_NAMES


def _truthy(a, x) -> bool:
    try:
        return bool(ir.evaluate(a, x))
    except ir.EvalError:
        return False


def sweep(accs, grid, block, max_instances: int = 2_000_000):
    """Brute force over every instance of every access (small launches)."""
    regions = sorted({a.record.region for a in accs})
    rank = {r: i for i, r in enumerate(regions)}
    # granule -> list of (is_read, access index, local, j, thread)
    cells: Dict[Tuple, List[Tuple]] = {}
    total = 0
    for ai, a in enumerate(accs):
        prog = a.program
        total += prog.instances
        if total > max_instances:
            raise ValueError("launch too large for the brute-force oracle")
        for local in range(prog.instances):
            x = None
            for k in range(prog.inner):
                y = prog.decode(local * prog.inner + k, prog.problem.nvars)
                if all(_truthy(at, y) for at in prog.path):
                    x = y
                    break
            if x is None:
                continue
            ids = tuple(int(x.get(n, prog.fixed.get(n, 0))) for n in ID_NAMES)
            off = ir.evaluate(prog.offset, x)
            shared = a.record.shared
            blk = (ids[2] * grid[1] + ids[1]) * grid[0] + ids[0]
            who = ids[3:] if shared else ids
            g = a.granule
            for j in range(a.record.width // g):
                byte = off + j * g
                cell = (rank[a.record.region], a.record.epoch if shared else 0,
                        blk if shared else 0, byte // g)
                cells.setdefault(cell, []).append(
                    (a.record.kind != "write", ai, local, j, who))
    racy = 0
    first = None
    for cell in sorted(cells):
        items = sorted(cells[cell], key=lambda t: (t[0], t[1], t[2], t[3]))
        head = items[0]
        if head[0]:
            continue                      # no write touches this granule
        other = next((t for t in items[1:] if t[4] != head[4]), None)
        if other is None:
            continue
        racy += 1
        if first is None:
            first = (cell, head, other)
    return racy > 0, racy, first
