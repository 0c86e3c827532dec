"""Concrete race replay with the specification's oracle semantics
(SPEC.md:573-631): read-write and write-write races
across instructions, with barrier epochs, over one concrete launch.

The reference's symbolic checker reports a DataRace only when a store races
with its own twin (engine/detectors.py:204-232: same instruction, equal
offsets, barriers ignored).  Its specification also defines a concrete
oracle -- not shipped with the reference -- that runs every (block, thread)
of a small launch, records an access trace (thread, region, byte offset,
width, read/write, barrier epoch) and pairs accesses "in the same region at
overlapping bytes from different threads with >= 1 write, same
barrier-epoch for shared memory, any epoch for global".
This module is that rule over the accesses the reference front end meets,
decided on the device by sorting (include/mk_b200.h mk_access_sweep).  It is
a NON-PARITY extension: ``GpuDetectors`` reports exactly the reference's
findings; this replay runs only when asked for.

Pipeline:
  1. ``AccessRecord``s come from ``GpuDetectors(record_accesses=True)``
     (every executed load / store on every explored path, with its path
     condition, byte offset, width, region and barrier epoch);
  2. each record becomes a path program at the launch
     (race.path_program with every thread id of the launch enumerated);
  3. per region a key layout (granule = gcd of the access widths; shared
     regions keyed by barrier epoch and block) so that equal keys are equal
     granules of one region;
  4. one device sweep: tuples, radix sort, segmented scan; the first race
     (least key) comes back as two dense tuple slots and is decoded here.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Mapping, Optional, Sequence, Tuple

from . import ir
from .compiler import _Ivl
from .race import ID_NAMES, NotSweepable, RaceProgram, path_program

KEY_LIMIT = 1 << 62
DIMS = ("gridDim.x", "gridDim.y", "gridDim.z", "blockDim.x", "blockDim.y", "blockDim.z")


@dataclass
class AccessRecord:
    """One executed access of one explored path (engine/executor.py:428-472):
    ``kind`` "read" (a load, or the read half of a compound store) or
    "write"; ``offset`` and ``path`` in the package IR."""

    kind: str
    line: int
    col: int
    text: str
    region: str
    shared: bool
    width: int
    offset: ir.Node
    path: List[ir.Node]
    epoch: int = 0


@dataclass
class Access:
    record: AccessRecord
    program: RaceProgram
    slot: int = 0        # first dense tuple slot
    tuples: int = 1      # tuples per instance
    granule: int = 1


@dataclass
class ReplayResult:
    has_race: bool
    racy: int                      # granules with a race
    instances: int
    tuples: int
    accesses: int                  # records swept
    skipped: List[Tuple[AccessRecord, str]] = field(default_factory=list)
    first: Optional[Dict] = None   # the first race: both accesses, threads, byte
    fast: bool = False             # decided by the owner-table pass (race-free)


def _threads(launch: Mapping[str, int]) -> Tuple[List[int], List[int]]:
    missing = [d for d in DIMS if d not in launch]
    if missing:
        raise NotSweepable(f"launch does not fix {missing}")
    return [int(launch[d]) for d in DIMS[:3]], [int(launch[d]) for d in DIMS[3:]]


def build(records: Sequence[AccessRecord], origin_of: Callable[[str], str],
          launch: Mapping[str, int], granule_one: Sequence[str] = ()):
    """Path programs and key layout of every sweepable record.  Returns
    (accesses, progs (mk_access_prog dicts), key_bits, skipped)."""
    grid, block = _threads(launch)
    ext = dict(zip(ID_NAMES, grid + block))
    accs: List[Access] = []
    skipped: List[Tuple[AccessRecord, str]] = []
    # every race has a write: a region no access writes (kernel inputs,
    # weights) cannot race, so its reads are never swept
    written = {r.region for r in records if r.kind == "write"}
    for r in records:
        if r.region not in written:
            continue
        try:
            prog = path_program(r.path, r.offset, r.shared, origin_of, launch, id_extents=ext)
        except NotSweepable as exc:
            skipped.append((r, str(exc)))
            continue
        accs.append(Access(r, prog))
    # offset range of every access (sound interval over its instance box)
    rng = []
    for a in accs:
        p = a.program.problem
        iv = _Ivl({n: (lo, hi) for n, lo, hi in zip(p.var_names, p.lo, p.hi)})(a.program.offset)
        if iv[0] is None or iv[1] is None:
            raise NotSweepable(f"unbounded offset at line {a.record.line}")
        rng.append(iv)
    nblocks = grid[0] * grid[1] * grid[2]
    regions: Dict[str, List[int]] = {}
    for i, a in enumerate(accs):
        regions.setdefault(a.record.region, []).append(i)
    progs: List[Dict] = [None] * len(accs)  # type: ignore[list-item]
    kbase = 0
    for rid in sorted(regions):
        idx = regions[rid]
        g = 0
        for i in idx:
            g = math.gcd(g, accs[i].record.width)
        if rid in granule_one or g < 1:
            g = 1
        lo = min(rng[i][0] for i in idx)
        lo = (lo // g) * g
        hi = max(rng[i][1] + accs[i].record.width for i in idx)
        span = -(-(hi - lo) // g)
        shared = accs[idx[0]].record.shared
        epochs = sorted({accs[i].record.epoch for i in idx}) if shared else [0]
        per_epoch = span * (nblocks if shared else 1)
        for i in idx:
            a = accs[i]
            a.granule = g
            a.tuples = a.record.width // g
            e = epochs.index(a.record.epoch) if shared else 0
            pr = a.program
            fixed = [int(pr.fixed.get(n, 0)) for n in ID_NAMES]
            progs[i] = {"off_reg": pr.off_reg, "n_exist": pr.n_exist, "id_var": list(pr.id_var),
                        "id_fixed": fixed, "write": 1 if a.record.kind == "write" else 0,
                        "shared": 1 if shared else 0, "granule": g, "tuples": a.tuples,
                        "kbase": kbase + e * per_epoch, "span": span, "off_lo": lo}
        kbase += per_epoch * len(epochs)
        if kbase >= KEY_LIMIT:
            raise NotSweepable("access keys exceed 62 bits")
    slot = 0
    for a in accs:
        a.slot = slot
        slot += a.program.instances * a.tuples
    key_bits = max(1, (max(kbase, 1) << 1).bit_length())
    return accs, progs, key_bits, skipped


def _locate(accs: Sequence[Access], slot: int) -> Tuple[Access, int, int]:
    lo, hi = 0, len(accs) - 1
    while lo < hi:
        m = (lo + hi + 1) // 2
        if accs[m].slot <= slot:
            lo = m
        else:
            hi = m - 1
    a = accs[lo]
    rel = slot - a.slot
    return a, rel // a.tuples, rel % a.tuples


def _thread_of(a: Access, x: Mapping[str, int]) -> Tuple[int, ...]:
    return tuple(int(x.get(n, a.program.fixed.get(n, 0))) for n in ID_NAMES)


def describe(a: Access, local: int, j: int) -> Dict:
    """One access instance: source position, kind, thread, byte."""
    prog = a.program
    x = prog.decode(local)
    if prog.n_exist:
        for k in range(prog.inner):
            y = prog.decode(local * prog.inner + k, prog.problem.nvars)
            if all(_truthy(at, y) for at in prog.path):
                x = y
                break
    byte = ir.evaluate(prog.offset, x) + j * a.granule
    return {"line": a.record.line, "col": a.record.col, "text": a.record.text,
            "kind": a.record.kind, "region": a.record.region, "epoch": a.record.epoch,
            "thread": _thread_of(a, x), "byte": byte}


def _truthy(at: ir.Node, x: Mapping[str, int]) -> bool:
    try:
        return bool(ir.evaluate(at, x))
    except ir.EvalError:
        return False


def replay_races(engine, records: Sequence[AccessRecord], origin_of: Callable[[str], str],
                 launch: Mapping[str, int]) -> ReplayResult:
    """Decide the oracle race rule for every recorded access at ``launch``
    on the device (``engine``: native.Engine)."""
    granule_one: List[str] = []
    for _ in range(2):
        accs, progs, key_bits, skipped = build(records, origin_of, launch, granule_one)
        if not accs:
            return ReplayResult(False, 0, 0, 0, 0, skipped)
        grid, block = _threads(launch)
        res = engine.access_sweep([a.program.problem for a in accs], progs, grid, block, key_bits,
                                  nkeys=1 << (key_bits - 1))
        if not res["misaligned"]:
            break
        # an offset not on its region's granule: byte granules everywhere
        granule_one = sorted({a.record.region for a in accs})
    else:  # pragma: no cover - granule 1 is always aligned
        raise RuntimeError("access sweep misaligned at granule 1")
    out = ReplayResult(bool(res["has_race"]), int(res["racy"]), int(res["instances"]),
                       int(res["tuples"]), len(accs), skipped, fast=bool(res.get("fast", 0)))
    if out.has_race:
        a, la, ja = _locate(accs, int(res["slot_a"]))
        b, lb, jb = _locate(accs, int(res["slot_b"]))
        out.first = {"write": describe(a, la, ja), "other": describe(b, lb, jb)}
    return out


def launch_model(checker, records: Sequence[AccessRecord], origin_of: Callable[[str], str],
                 pins: Mapping[str, int]) -> Dict[str, int]:
    """A concrete launch for a replay: the canonical model (decided by the
    engine, ``checker``: engine.SiteChecker) of the launch-level atoms of the
    first recorded path -- the context's initial constraints and wrapper
    facts (engine/executor.py:152-200) -- with ``pins`` (e.g. BS, SL) fixed."""
    from .race import THREAD_PRIVATE

    path = records[0].path
    widths: Dict[str, str] = {}
    for a in path:
        ir.symbols_of(a, widths)
    atoms = [a for a in path
             if all(origin_of(n) not in THREAD_PRIVATE for n in ir.symbols_of(a))]
    for k, v in pins.items():
        w = widths.get(k, "i64")
        atoms.append(("p", "eq", ("s", k, w), ("c", int(v), w)))
    r = checker.check(atoms, origin_of)
    if r.status != "sat":
        raise NotSweepable(f"no launch with {dict(pins)}: {r.status}")
    return dict(r.witness)
