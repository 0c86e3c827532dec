"""Drop-in replacement of the reference checker ``Detectors``.

The reference checking stage is ``minikernel.engine.detectors.Detectors``
(engine/detectors.py:46-57), constructed by the executor as
``Detectors(self.solver, self.table, self.kernel.name, detector_options)``
(engine/executor.py:116-117) and called at five sites
(engine/executor.py:376, 407, 432/434, 468-472).  ``GpuDetectors`` keeps that
constructor, the public fields (``findings``, ``enabled``), the per-site memo,
the overflow cascade, the ``flagged_io`` side effects and the exact query each
site builds; only the decision and the canonical witness come from the B200
engine instead of ``Solver.check`` + ``canonicalize_witness``
(engine/report.py:147-174).

Install it with :func:`install` (rebinds the name the executor resolves,
engine/executor.py:33) or pass it around explicitly.  The host-side rules are
restated from the reference, file:line cited per method.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

from . import ir
from .engine import QueryResult, SiteChecker

_SHARED: Dict[int, SiteChecker] = {}
_LOCK = threading.Lock()


def shared_checker(device: int = 0) -> SiteChecker:
    """One engine context per device, reused across analyses."""
    with _LOCK:
        chk = _SHARED.get(device)
        if chk is None:
            chk = SiteChecker(device=device)
            _SHARED[device] = chk
        return chk


def _ref():
    """The reference modules the checker API is defined in (imported lazily:
    the drop-in lives inside a process that already runs the reference)."""
    from minikernel.engine import report as R
    from minikernel.engine import state as S
    from minikernel.sym import expr as E
    from minikernel import tensor as T
    return E, R, S, T


@dataclass
class GpuDetectors:
    """Same constructor, fields and site methods as the reference
    ``Detectors`` (engine/detectors.py:46-57)."""

    solver: object
    table: object
    kernel: str
    options: object = None
    findings: List[object] = field(default_factory=list)
    enabled: bool = True
    _memo: Dict[Tuple[str, int, int], bool] = field(default_factory=dict)
    device: int = 0
    checker: Optional[SiteChecker] = None
    _cache: Dict[Tuple[str, ...], QueryResult] = field(default_factory=dict)
    _screen_cache: Dict[Tuple[str, ...], str] = field(default_factory=dict)
    screens: int = 0                  # screening queries decided on the device
    screen_budget_unknowns: int = 0   # of those, cut off by the per-query budget
    # non-parity: record every executed access for the oracle race replay
    # (paper_2603_24595_b200.replay); off by default
    record_accesses: bool = False
    accesses: List[object] = field(default_factory=list)
    # (kind, line, col) -> IR assertions of the first sat query of the site,
    # for witness replay (paper_2603_24595_b200.witness); off by default
    record_queries: bool = False
    sat_queries: Dict[Tuple[str, int, int], List[object]] = field(default_factory=dict)

    def __post_init__(self) -> None:
        if self.options is None:
            from minikernel.engine.detectors import DetectorOptions
            self.options = DetectorOptions()
        if self.checker is None:
            self.checker = shared_checker(self.device)
        self._query_ir: Dict[Tuple[str, ...], List[object]] = {}
        self._last_query = None
        E, R, S, T = _ref()
        self._E, self._R, self._S, self._T = E, R, S, T
        lo, hi = E.I32.bounds()
        self._i32 = (lo, hi)

    # -- shared decision path ------------------------------------------------

    def _decide(self, assertions) -> QueryResult:
        """Decide one query on the B200 engine.  Identical queries share one
        verdict, as the reference's render-keyed solver cache does
        (solver/interface.py:54-60)."""
        E = self._E
        key = tuple(E.render(a) for a in assertions)
        got = self._cache.get(key)
        if got is not None:
            if self.record_queries:
                self._last_query = self._query_ir.get(key)
            return got
        q = [ir.from_ref(a) for a in assertions]
        res = self.checker.check(q, self.table.origin_of)
        self._cache[key] = res
        if self.record_queries:
            self._query_ir[key] = q
            self._last_query = q
        return res

    def _status(self, state, key) -> str:
        """engine/detectors.py:59-65: findings on an undecided path are
        honest unknowns; only clean proofs feed the per-site memo."""
        if state.unknown_path:
            return "unknown"
        self._memo[key] = True
        return "sat"

    def _emit(self, kind, line, col, text, blamed, res, state, key, region=None,
              offset=None, flag_node=None) -> None:
        Finding = self._R.Finding
        if res.status == "sat":
            if self.record_queries and key not in self.sat_queries and self._last_query:
                self.sat_queries[key] = self._last_query
            status = self._status(state, key)
            if flag_node is not None:
                state.flagged_io.append(flag_node)
            self.findings.append(Finding(
                kind=kind, kernel=self.kernel, line=line, column=col, blamed_text=text,
                blamed_expr=blamed, status=status, witness=dict(res.witness),
                region=region, offset_expr=offset))
        elif res.status == "unknown":
            self.findings.append(Finding(
                kind=kind, kernel=self.kernel, line=line, column=col, blamed_text=text,
                blamed_expr=blamed, status="unknown", region=region, offset_expr=offset))

    # -- IntegerOverflow (engine/detectors.py:69-130) --------------------------

    def arithmetic_site(self, state, node, line: int, col: int, text: str) -> None:
        E = self._E
        if not (self.enabled and self.options.check_overflow):
            return
        if not isinstance(node, E.BinOp) or node.op not in ("add", "mul", "shl"):
            return
        if node.width == E.I32:
            lo, hi = self._i32
        elif node.width == E.U32 and self.options.check_unsigned_wrap:
            lo, hi = E.U32.bounds()
        else:
            return
        self._overflow(state, node, node, lo, hi, line, col, text)

    def narrowing_site(self, state, node, line: int, col: int, text: str) -> None:
        if not (self.enabled and self.options.check_overflow and self.options.check_narrowing):
            return
        if node.width.is_float or node.arg.width.is_float:
            return
        if node.width.bits >= node.arg.width.bits:
            return
        lo, hi = node.width.bounds()
        self._overflow(state, node, node.arg, lo, hi, line, col, text)

    def _overflow(self, state, blamed, value, lo: int, hi: int, line, col, text) -> None:
        E = self._E
        kids = E.children(blamed)
        if any(E.contains(k, prior) for prior in state.flagged_io for k in kids):
            return  # cascade of an already flagged overflow
        key = ("IntegerOverflow", line, col)
        if self._memo.get(key):
            state.flagged_io.append(blamed)
            return
        itv = E.interval(value)
        if itv[0] is not None and itv[1] is not None and lo <= itv[0] and itv[1] <= hi:
            return
        escape = E.BoolOp("or", (E.Cmp("gt", value, E.Const(hi, E.I64)),
                                 E.Cmp("lt", value, E.Const(lo, E.I64))))
        res = self._decide(state.path + [escape])
        self._emit("IntegerOverflow", line, col, text, blamed, res, state, key,
                   flag_node=blamed)

    # -- OutOfBounds (engine/detectors.py:134-200) ---------------------------------

    def access_site(self, state, addr, nbytes: int, line: int, col: int, text: str) -> None:
        E = self._E
        if not self.enabled or not addr.known:
            return
        if self.record_accesses:
            self._record(state, addr, nbytes, line, col, text)
        key = ("OutOfBounds", line, col)
        if self._memo.get(key):
            return
        query = state.path + [E.not_(self._T.in_bounds(addr, nbytes))]
        query.extend(self._pin(n) for n in self._overflow_nodes(addr.offset_bytes))
        res = self._decide(query)
        self._emit("OutOfBounds", line, col, text, addr.offset_bytes, res, state, key,
                   region=addr.provenance.rid, offset=addr.offset_bytes)

    def _overflow_nodes(self, root) -> list:
        """Every node the overflow checks would examine, in the reference's
        pre-order stack walk (engine/detectors.py:166-186)."""
        E = self._E
        if not self.options.check_overflow:
            return []
        out, todo = [], [root]
        while todo:
            e = todo.pop()
            todo.extend(E.children(e))
            if isinstance(e, E.BinOp) and e.op in ("add", "mul", "shl"):
                if e.width == E.I32 or (e.width == E.U32 and self.options.check_unsigned_wrap):
                    out.append(e)
            elif isinstance(e, E.Cast) and self.options.check_narrowing \
                    and not e.width.is_float and not e.arg.width.is_float \
                    and e.width.bits < e.arg.width.bits:
                out.append(e)
        return out

    def _pin(self, node):
        """Keep a node inside its width (engine/detectors.py:188-200)."""
        E = self._E
        lo, hi = node.width.bounds()
        value = node.arg if isinstance(node, E.Cast) else node
        return E.and_(E.Cmp("ge", value, E.Const(lo, E.I64)),
                      E.Cmp("le", value, E.Const(hi, E.I64)))

    # -- DataRace (engine/detectors.py:204-273) -------------------------------------

    def _record(self, state, addr, nbytes, line, col, text) -> None:
        """An executed access (engine/executor.py:428-472) with its path
        condition and barrier epoch (engine/state.py:142); the store that
        follows turns it into a write (store_site)."""
        from .replay import AccessRecord

        region = addr.provenance
        self.accesses.append(AccessRecord(
            kind="read", line=line, col=col, text=text, region=region.rid,
            shared=region.kind == "shared", width=int(nbytes),
            offset=ir.from_ref(addr.offset_bytes), path=[ir.from_ref(a) for a in state.path],
            epoch=int(getattr(state, "barrier_epoch", 0))))
        self._last_access = (id(state), line, col, addr.offset_bytes)

    def store_site(self, state, region, addr, nbytes: int, line: int, col: int,
                   text: str) -> None:
        E = self._E
        if self.record_accesses and self.enabled and self.accesses and \
                getattr(self, "_last_access", None) == (id(state), line, col, addr.offset_bytes):
            self.accesses[-1].kind = "write"
        if not self.enabled or state.thread is None:
            return
        key = ("DataRace", line, col)
        if self._memo.get(key):
            return
        offset = addr.offset_bytes
        twin = self._twins(state, offset)
        query = state.path + [E.substitute(p, twin) for p in state.path]
        query.append(E.Cmp("eq", offset, E.substitute(offset, twin)))
        query.append(self._distinct(state.thread, twin, region.kind == "shared"))
        res = self._decide(query)
        self._emit("DataRace", line, col, text, offset, res, state, key,
                   region=region.rid, offset=offset)

    def _twins(self, state, offset) -> Dict[str, object]:
        """Prime every thread-private symbol of the path and the offset."""
        E = self._E
        pool: Dict[str, object] = {}
        for p in state.path:
            pool.update(E.symbols_of(p))
        pool.update(E.symbols_of(offset))
        private = self._S.THREAD_PRIVATE
        return {n: E.Sym(n + "'", s.width) for n, s in pool.items()
                if self.table.origin_of(n) in private}

    def _distinct(self, thread, twin, shared: bool):
        """Distinct twin identities; shared memory also requires the same
        block."""
        E = self._E
        same = lambda s: E.Cmp("eq", s, twin.get(s.name, s))  # noqa: E731
        blocks = [same(thread.block_idx[a]) for a in self._S.AXES]
        threads = [same(thread.thread_idx[a]) for a in self._S.AXES]
        if shared:
            return E.and_(*(blocks + [E.not_(E.and_(*threads))]))
        return E.not_(E.and_(*(blocks + threads)))

    # -- InvalidDeref (engine/detectors.py:277-298) ---------------------------------

    def deref_site(self, state, addr, line: int, col: int, text: str) -> None:
        if not self.enabled or addr.known:
            return
        key = ("InvalidDeref", line, col)
        if self._memo.get(key):
            return
        res = self._decide(list(state.path))
        self._emit("InvalidDeref", line, col, text, addr.offset_bytes, res, state, key)


    # -- branch screening (engine/executor.py:489-492), SURVEY.md 8(f) row 1 --

    # the reference grants every solver query, screening included, its own
    # Budget.query_timeout_s (engine/state.py:38; solver/interface.py:21-28)
    SCREEN_BUDGET_S = 30.0

    def screen(self, path, cond) -> str:
        """sat | unsat | unknown for path + cond, as the executor's
        ``_screen`` (engine/executor.py:489-492): feasibility only (the engine
        stops at the first model, MK_PF_ANY), render-keyed cache like
        ``Solver.check`` (solver/interface.py:54-60).  Decided on the B200
        only: there is no host or reference fallback.  A screen the device
        cannot finish within the reference's per-query timeout is
        ``unknown``, exactly as a reference timeout would be, and is counted
        in ``screen_budget_unknowns``."""
        E = self._E
        assertions = list(path) + [cond]
        key = ("screen",) + tuple(E.render(a) for a in assertions)
        got = self._screen_cache.get(key)
        if got is None:
            res = self.checker.feasible([ir.from_ref(a) for a in assertions],
                                        self.table.origin_of, max_seconds=self.SCREEN_BUDGET_S)
            got = res.status
            self.screens += 1
            if got == "unknown" and res.reason == "budget":
                self.screen_budget_unknowns += 1
            self._screen_cache[key] = got
        return got


def install(device: int = 0, checker: Optional[SiteChecker] = None, screening: bool = False,
            recorders: Optional[list] = None, created: Optional[list] = None,
            record_queries: bool = False):
    """Swap the checking stage of the reference executor for the B200 engine
    (engine/executor.py:33 resolves ``Detectors`` at construction time); with
    ``screening`` the executor's branch screening (engine/executor.py:489-492)
    also runs on the engine.  With ``recorders`` (a list) every constructed
    detector also records the executed accesses for the oracle race replay
    (paper_2603_24595_b200.replay) and is appended to it.  Returns what
    ``uninstall`` needs to restore.  ``created`` (a list) collects every
    detector the executor constructs (screening counters)."""
    import minikernel.engine.executor as X

    prev = (X.Detectors, X.Executor._screen)

    class _Bound(GpuDetectors):
        def __init__(self, solver, table, kernel, options=None):
            super().__init__(solver, table, kernel, options, device=device, checker=checker,
                             record_accesses=recorders is not None,
                             record_queries=record_queries)
            if recorders is not None:
                recorders.append(self)
            if created is not None:
                created.append(self)

    _Bound.__name__ = "GpuDetectors"
    X.Detectors = _Bound
    if screening:
        orig = prev[1]

        def _screen(self, state, cond):
            det = getattr(self, "detectors", None)
            if isinstance(det, GpuDetectors):
                return det.screen(state.path, cond)
            return orig(self, state, cond)

        X.Executor._screen = _screen
    return prev


def uninstall(prev) -> None:
    import minikernel.engine.executor as X

    if isinstance(prev, tuple):
        X.Detectors, X.Executor._screen = prev
    else:
        X.Detectors = prev
