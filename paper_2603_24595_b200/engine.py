"""Checking-stage facade: compile site queries, decide them on the device,
assemble the reference-format verdicts.

``check_queries`` is the batch entry point (one device call for any number
of sites); ``SiteChecker.check`` is the single-query path used by the
drop-in detectors.  Both return, per query, ``(status, witness)`` with the
reference's meaning: ``sat`` + canonical witness (engine/report.py:147-174),
``unsat``, or ``unknown`` (solver/query.py:11-42).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import ir
from .compiler import CompileError, CompiledQuery, compile_query
from .native import Engine, PackedSet

DEFAULT_LIMITS = {"max_seconds": 30.0}   # Budget.query_timeout_s (engine/state.py:38)


@dataclass
class QueryResult:
    status: str
    witness: Dict[str, int]
    reason: Optional[str] = None


@dataclass
class BatchStats:
    queries: int = 0
    problems: int = 0
    compile_s: float = 0.0
    device_s: float = 0.0
    assemble_s: float = 0.0
    device: Dict[str, float] = field(default_factory=dict)


def compile_all(queries: Sequence[Tuple[Sequence[ir.Node], Callable[[str], str]]]
                ) -> List[Tuple[Optional[CompiledQuery], Optional[str]]]:
    out = []
    for assertions, origin_of in queries:
        try:
            out.append((compile_query(assertions, origin_of), None))
        except CompileError as exc:
            out.append((None, str(exc)))
    return out


class SiteChecker:
    """Holds one device context; decides compiled queries in batches."""

    def __init__(self, device: int = 0, lib_path: Optional[str] = None,
                 limits: Optional[dict] = None) -> None:
        self.engine = Engine(device, lib_path)
        self.limits = dict(DEFAULT_LIMITS)
        if limits:
            self.limits.update(limits)
        self.stats = BatchStats()

    def close(self) -> None:
        self.engine.close()

    def pack(self, compiled: Sequence[Optional[CompiledQuery]]) -> Tuple[PackedSet, List[int]]:
        problems, offsets = [], []
        for cq in compiled:
            offsets.append(len(problems))
            if cq is not None:
                problems.extend(cq.problems)
        return PackedSet(problems), offsets

    def decide(self, compiled: Sequence[Tuple[Optional[CompiledQuery], Optional[str]]],
               packed: Optional[PackedSet] = None, offsets: Optional[List[int]] = None
               ) -> List[QueryResult]:
        cqs = [c for c, _ in compiled]
        if packed is None:
            packed, offsets = self.pack(cqs)
        t0 = time.perf_counter()
        # the reference grants every query its own timeout (engine/state.py:38);
        # a batch gets the sum, capped
        lim = dict(self.limits)
        lim["max_seconds"] = min(self.limits["max_seconds"] * max(len(compiled), 1), 3600.0)
        results = self.engine.solve_packed(packed, lim) if packed.problems else []
        t1 = time.perf_counter()
        out: List[QueryResult] = []
        for (cq, err), off in zip(compiled, offsets):
            if cq is None:
                out.append(QueryResult("unknown", {}, err))
                continue
            res = results[off:off + len(cq.problems)]
            status, witness = cq.assemble(res)
            out.append(QueryResult(status, witness))
        t2 = time.perf_counter()
        self.stats.queries += len(compiled)
        self.stats.problems += len(packed.problems)
        self.stats.device_s += t1 - t0
        self.stats.assemble_s += t2 - t1
        if self.engine.last_stats:
            for k, v in self.engine.last_stats.items():
                self.stats.device[k] = self.stats.device.get(k, 0) + v
        return out

    def check_queries(self, queries: Sequence[Tuple[Sequence[ir.Node], Callable[[str], str]]]
                      ) -> List[QueryResult]:
        t0 = time.perf_counter()
        compiled = compile_all(queries)
        self.stats.compile_s += time.perf_counter() - t0
        return self.decide(compiled)

    def check(self, assertions: Sequence[ir.Node], origin_of: Callable[[str], str]) -> QueryResult:
        return self.check_queries([(assertions, origin_of)])[0]
