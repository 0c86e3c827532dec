"""Multi-GPU checking: one process per GPU (torch.distributed), two ways to
split the work.

``check_corpus``  -- kernel x model sweep (BASELINE.json configs[4]): every
    corpus entry (one kernel port under one model context, i.e. one site set)
    is an independent unit; entries are dealt to ranks by estimated cost and
    each rank decides its own entries with no data-path collective.  One
    ``all_gather_object`` hands every rank the full result list at the end.

``check_sites``  -- one site set, the sites dealt to ranks (each site is an
    independent query); one ``all_gather_object`` of the verdict records.

``check_slabbed`` -- one site set, every problem's root box cut into
    ``world`` slabs along its first splittable symbol; rank r searches slab r
    (so one hard query uses every GPU).  The per-problem results are combined
    exactly: the canonical witness is the lexicographic optimum, in witness
    order, over the slabs' optima (engine/report.py:147-203), ``unknown`` if
    any slab is undecided, ``unsat`` if every slab is.  The combination is a
    single all-gather of a fixed-width int64 record per problem (status +
    128-bit point words), an NCCL collective over NVLink on the GPU path and
    gloo in the CPU tests.

Both entry points reuse one ``SiteChecker`` per rank; on the GPU path the
checker is bound to ``cuda:<local_rank>``.
"""

from __future__ import annotations

import dataclasses
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import ir
from .compiler import CompiledQuery, Problem
from .engine import QueryResult, SiteChecker

Query = Tuple[Sequence[ir.Node], Callable[[str], str]]

# "giveup": undecided for a reason other than the budget (an overflow or
# engine limit) -- unknown in the result, never searched again
_STATUS = {"unsat": 0, "sat": 1, "unknown": 2, "giveup": 3}
_STATUS_NAME = {v: k for k, v in _STATUS.items()}
_MASK64 = (1 << 64) - 1


def _dist():
    import torch.distributed as dist

    return dist


def _world(group=None) -> Tuple[int, int]:
    dist = _dist()
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


# -- corpus sharding --------------------------------------------------------------------

def entry_cost(queries: Sequence[Query]) -> float:
    """Static cost estimate of one corpus entry (sites x atoms), used only to
    balance the deal; any estimate gives the same results."""
    return float(sum(1 + len(a) for a, _ in queries))


def deal(costs: Sequence[float], world: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of entries to ranks."""
    loads = [0.0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda k: (loads[k], k))
        out[r].append(i)
        loads[r] += costs[i]
    for lst in out:
        lst.sort()
    return out


def check_corpus(checker: SiteChecker, entries: Sequence[Sequence[Query]], group=None
                 ) -> List[List[QueryResult]]:
    """Decide every entry of a kernel x model corpus across the ranks of
    ``group``; every rank returns the full, ordered result list."""
    rank, world = _world(group)
    mine = deal([entry_cost(e) for e in entries], world)[rank]
    local: Dict[int, List[QueryResult]] = {}
    for i in mine:
        local[i] = checker.check_queries(entries[i])
    if world == 1:
        return [local[i] for i in range(len(entries))]
    dist = _dist()
    gathered: List[Optional[Dict[int, List[QueryResult]]]] = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    merged: Dict[int, List[QueryResult]] = {}
    for part in gathered:
        merged.update(part or {})
    return [merged[i] for i in range(len(entries))]


def check_sites(checker: SiteChecker, queries: Sequence[Query], group=None
                ) -> List[QueryResult]:
    """Decide one site set across the ranks of ``group``: sites are
    independent queries (each is one ``Solver.check`` + canonicalisation in
    the reference, engine/detectors.py:111-130), dealt longest-first by
    assertion count; each rank compiles and decides its share in one device
    batch, and one ``all_gather_object`` of the (index, verdict, witness)
    records gives every rank the ordered result list.  No data-path
    collective: the records are a few KB."""
    rank, world = _world(group)
    if world == 1:
        return checker.check_queries(queries)
    mine = deal([float(1 + len(a)) for a, _ in queries], world)[rank]
    got = checker.check_queries([queries[i] for i in mine]) if mine else []
    local = {i: (r.status, r.witness, r.reason) for i, r in zip(mine, got)}
    dist = _dist()
    gathered: List[Optional[Dict[int, tuple]]] = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    merged: Dict[int, tuple] = {}
    for part in gathered:
        merged.update(part or {})
    return [QueryResult(*merged[i]) for i in range(len(queries))]


# -- slab sharding ----------------------------------------------------------------------

def slab(p: Problem, rank: int, world: int) -> Optional[Problem]:
    """The rank-th of ``world`` slabs of ``p``'s root box along its first
    symbol (witness order) with at least two values, pieces ordered best
    first in that symbol's direction; None when the slab is empty."""
    v = next((i for i in range(p.nvars) if p.hi[i] > p.lo[i]), None)
    if v is None:
        return p if rank == 0 else None
    size = p.hi[v] - p.lo[v] + 1
    q, rem = divmod(size, world)
    j = (world - 1 - rank) if p.maximize[v] else rank   # ascending piece index
    start = j * q + min(j, rem)
    length = q + (1 if j < rem else 0)
    if length <= 0:
        return None
    lo, hi = list(p.lo), list(p.hi)
    lo[v] = p.lo[v] + start
    hi[v] = lo[v] + length - 1
    return dataclasses.replace(p, lo=lo, hi=hi)


def _better(x: Sequence[int], y: Sequence[int], maximize: Sequence[bool]) -> bool:
    for a, b, mx in zip(x, y, maximize):
        if a != b:
            return a > b if mx else a < b
    return False


def combine_slabs(problems: Sequence[Problem],
                  per_rank: Sequence[Sequence[Tuple[str, Optional[List[int]]]]]
                  ) -> List[Tuple[str, Optional[List[int]]]]:
    """Exact combination of the slab results of every problem."""
    out = []
    for k, p in enumerate(problems):
        rs = [r[k] for r in per_rank]
        if any(s in ("unknown", "giveup") for s, _ in rs):
            out.append(("unknown", None))
            continue
        best = None
        for s, pt in rs:
            if s == "sat" and (best is None or _better(pt, best, p.maximize)):
                best = pt
        out.append(("sat", list(best)) if best is not None else ("unsat", None))
    return out


def _encode(problems: Sequence[Problem], results) -> List[int]:
    rec: List[int] = []
    for p, (s, pt) in zip(problems, results):
        rec.append(_STATUS[s])
        vals = pt if pt is not None else [0] * p.nvars
        for v in vals:
            rec.append(v & _MASK64)          # low word
            rec.append(v >> 64)              # high word (signed)
    return rec


def _decode(problems: Sequence[Problem], rec: Sequence[int]):
    out, i = [], 0
    for p in problems:
        s = _STATUS_NAME[int(rec[i])]
        i += 1
        pt = []
        for _ in range(p.nvars):
            lo, hi = int(rec[i]) & _MASK64, int(rec[i + 1])
            pt.append((hi << 64) | lo)
            i += 2
        out.append((s, pt if s == "sat" else None))
    return out


def _all_gather_records(rec: List[int], device, group=None) -> List[List[int]]:
    import torch

    dist = _dist()
    _, world = _world(group)
    # int64 words: the low 64-bit halves travel as their two's complement
    words = [w - (1 << 64) if w >= (1 << 63) else w for w in rec]
    t = torch.tensor(words, dtype=torch.int64, device=device)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return [[int(x) for x in o.cpu().tolist()] for o in outs]


def slab_rounds(total_s: float, first_s: float = 0.25) -> List[float]:
    """Budget of each exchange round of ``check_slabbed``: doubling slices
    from ``first_s`` whose sum is ``total_s`` (the same schedule on every
    rank, so every rank enters the same number of collectives)."""
    out: List[float] = []
    left, cur = float(total_s), float(first_s)
    while left > 1e-9:
        t = min(cur, left)
        out.append(t)
        left -= t
        cur *= 2.0
    return out or [float(total_s)]


def dominated(p: Problem, rank: int, statuses: Sequence[str]) -> bool:
    """Slab ``rank`` of ``p`` cannot hold the combined answer once another
    slab has a model: slabs are ordered best first along the first symbol
    with two values (every earlier symbol is fixed), so every point of a
    lower slab precedes every point of this one in witness order; for a
    feasibility-only problem any model decides."""
    if p.any_model:
        return any(s == "sat" for r, s in enumerate(statuses) if r != rank)
    return any(s == "sat" for s in statuses[:rank])


def check_slabbed(checker: SiteChecker, queries: Sequence[Query], group=None,
                  device=None, first_round_s: float = 0.25) -> List[QueryResult]:
    """Decide one site set with every problem's root box split across the
    ranks of ``group``; every rank returns the same results.

    The search runs in rounds of doubling budget (``slab_rounds``).  After
    each round the ranks exchange their per-problem results (one all-gather
    of fixed-width records): a slab still undecided on one rank stops as soon
    as a better-ordered slab has a model (``dominated``), i.e. the incumbents
    are shared at round boundaries; only the slabs still open are searched
    again, with twice the budget.  Without budget cut-offs the result is the
    exact combination (``combine_slabs``) of every slab's optimum."""
    rank, world = _world(group)
    compiled = checker.compile(queries)
    problems: List[Problem] = []
    offsets: List[int] = []
    for cq, _ in compiled:
        offsets.append(len(problems))
        if cq is not None:
            problems.extend(cq.problems)
    mine = [slab(p, rank, world) for p in problems]
    local: List[Tuple[str, Optional[List[int]]]] = [
        ("unsat", None) if m is None else ("unknown", None) for m in mine]
    live = [k for k, m in enumerate(mine) if m is not None]
    total = min(checker.limits["max_seconds"] * max(len(queries), 1), 3600.0)
    if world > 1 and device is None:
        # NCCL only moves device tensors; gloo (the CPU tests) host ones
        import torch

        nccl = _dist().get_backend(group) == "nccl"
        device = f"cuda:{torch.cuda.current_device()}" if nccl else "cpu"
    per_rank = [local]
    self_rounds = 0
    for budget in slab_rounds(total, first_round_s):
        if live:
            lim = dict(checker.limits)
            lim["max_seconds"] = budget
            solved = checker.engine.solve([mine[k] for k in live], lim)
            # a call that ended well inside its budget did not cut anything
            # off: its unknowns are give-ups, not worth a longer round
            cut = checker.engine.last_stats.get("seconds", budget) >= 0.5 * budget
            for k, r in zip(live, solved):
                local[k] = r if (r[0] != "unknown" or cut) else ("giveup", None)
        self_rounds += 1
        if world > 1:
            recs = _all_gather_records(_encode(problems, local), device, group)
            per_rank = [_decode(problems, r) for r in recs]
        else:
            per_rank = [local]
        # open = undecided here and not dominated by another slab's model
        # (computed from the gathered records: the same on every rank)
        open_any = False
        for k, p in enumerate(problems):
            sts = [pr[k][0] for pr in per_rank]
            for r in range(world):
                if sts[r] == "unknown" and dominated(p, r, sts):
                    sts[r] = "unsat"          # nothing here beats the better slab
                    per_rank[r][k] = ("unsat", None)
            if "unknown" in sts:
                open_any = True
        local[:] = per_rank[rank]
        live = [k for k in live if local[k][0] == "unknown"]
        if not open_any:
            break
    checker.last_slab_rounds = self_rounds
    results = combine_slabs(problems, per_rank)
    out: List[QueryResult] = []
    for (cq, err), off in zip(compiled, offsets):
        if cq is None:
            out.append(QueryResult("unknown", {}, err))
            continue
        status, witness = cq.assemble(results[off:off + len(cq.problems)])
        out.append(QueryResult(status, witness))
    return out


# -- K2 race sweep across GPUs ------------------------------------------------------------

def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous instance range of one rank (instance order = key order for
    the fused pass, so shards meet at one boundary pair each)."""
    return total * rank // world, total * (rank + 1) // world


def combine_race_shards(parts: Sequence[dict]) -> Optional[dict]:
    """Exact combination of ranged sweeps in rank order: conflicts inside
    each shard plus one boundary pair per pair of adjacent non-empty shards
    (the last access of one and the first of the next: equal key, distinct
    identity); the first conflict is the least (idx_b << 32 | idx_a).  None
    when a shard or a boundary is out of key order (the fused pass does not
    apply: the launch is swept whole)."""
    if any(not p["sorted"] for p in parts):
        return None
    out = {"instances": sum(p["instances"] for p in parts),
           "tuples": sum(p["tuples"] for p in parts),
           "conflicts": sum(p["conflicts"] for p in parts), "sorted": 1, "fused": 1}
    cands = [((p["idx_b"] << 32) | p["idx_a"], p["offset"]) for p in parts if p["has_race"]]
    prev = None
    for p in parts:
        if not p["have"]:
            continue
        if prev is not None:
            if p["first_key"] < prev["last_key"]:
                return None
            if p["first_key"] == prev["last_key"] and p["first_id"] != prev["last_id"]:
                out["conflicts"] += 1
                cands.append(((p["first_idx"] << 32) | prev["last_idx"],
                              p["first_key"] // p["nblocks"] + p["off_lo"]))
        prev = p
    out["has_race"] = int(out["conflicts"] > 0)
    if cands:
        c, off = min(cands)
        out["idx_b"], out["idx_a"], out["offset"] = c >> 32, c & 0xffffffff, off
    else:
        out["idx_a"] = out["idx_b"] = out["offset"] = 0
    return out


def race_sweep_sharded(engine, prog, group=None) -> dict:
    """K2 over every rank: rank r sweeps its contiguous
    instance range with the fused ordered pass; one all_gather_object of the
    per-shard summaries (a few hundred bytes) and the exact combination give
    every rank the result the single-GPU sweep returns.  If any shard's keys
    (or a shard boundary) are out of order, rank 0 sweeps the whole launch
    (radix-sort path) and broadcasts its result."""
    rank, world = _world(group)
    keys = ("instances", "tuples", "conflicts", "has_race", "idx_a", "idx_b", "offset", "sorted")
    if world == 1:
        return engine.race_sweep(prog)
    dist = _dist()
    b, e = shard_range(prog.instances, rank, world)
    mine = engine.race_sweep(prog, b, e) if e > b else \
        {"sorted": 1, "have": 0, "instances": 0, "tuples": 0, "conflicts": 0, "has_race": 0}
    mine = {k: v for k, v in mine.items() if k != "pair"}
    parts: List[dict] = [None] * world  # type: ignore[list-item]
    dist.all_gather_object(parts, mine, group=group)
    got = combine_race_shards(parts)
    if got is None:
        box = [engine.race_sweep(prog) if rank == 0 else None]
        if box[0] is not None:
            box[0] = {k: box[0][k] for k in keys}
        dist.broadcast_object_list(box, src=0, group=group)
        got = box[0]
    if got["has_race"]:
        got["pair"] = (prog.decode(got["idx_a"]), prog.decode(got["idx_b"]))
    return got
