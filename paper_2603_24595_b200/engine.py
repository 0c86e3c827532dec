"""Checking-stage facade: compile site queries, decide them on the device,
assemble the reference-format verdicts.

``check_queries`` is the batch entry point (one device call for any number
of sites); ``SiteChecker.check`` is the single-query path used by the
drop-in detectors.  Both return, per query, ``(status, witness)`` with the
reference's meaning: ``sat`` + canonical witness (engine/report.py:147-174),
``unsat``, or ``unknown`` (solver/query.py:11-42).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import ir
from .compiler import CapacityError, CompileError, CompiledQuery, compile_query
from .native import Engine, PackedSet
from .order import OriginLookup

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
    tier1_decided: int = 0         # queries decided by the light first tier
    tier2_queries: int = 0         # queries that went through the full presolve
    tier1_batches: int = 0         # device calls of the first tier
    tier1_s: float = 0.0           # wall time of those calls
    tier2_batches: int = 0
    tier2_s: float = 0.0
    device_s: float = 0.0
    assemble_s: float = 0.0
    device: Dict[str, float] = field(default_factory=dict)


LIGHT_FAILED = "light compile: left to the full presolve"


def _compile_one(item) -> Tuple[Optional[CompiledQuery], Optional[str]]:
    """(assertions, origin lookup[, light]) -> (compiled query, error).  A
    light compile that hits an engine limit (typically a symbol only the full
    presolve bounds) is not an error: the query goes to the second tier."""
    assertions, origin_of = item[0], item[1]
    light = len(item) > 2 and bool(item[2])
    t0 = time.perf_counter()
    try:
        cq = compile_query(assertions, origin_of, light)
        cq.compile_s = time.perf_counter() - t0
        return cq, None
    except CompileError as exc:
        return None, (LIGHT_FAILED if light else str(exc))
    except CapacityError:
        if light:
            return None, LIGHT_FAILED
        raise


def compile_all(queries: Sequence[Tuple[Sequence[ir.Node], Callable[[str], str]]],
                light: bool = False) -> List[Tuple[Optional[CompiledQuery], Optional[str]]]:
    return [_compile_one((q[0], q[1], light)) for q in queries]


def _portable(query):
    """(assertions, origin map) with a picklable origin lookup."""
    assertions, origin_of = query
    if isinstance(origin_of, OriginLookup):
        return assertions, origin_of
    names: Dict[str, str] = {}
    for a in assertions:
        ir.symbols_of(a, names)
    return assertions, OriginLookup({n.rstrip("'"): origin_of(n) for n in names})


class CompilePool:
    """Host-side site compilation across worker processes.

    Sites are independent, so a batch of queries is compiled in parallel on
    the host cores (the compiler is pure Python; one process per core side
    steps the GIL).  The workers are fresh interpreters
    (``python -m paper_2603_24595_b200.compile_worker``) started once per
    checker, never forks of the checker's process: a fork would copy the
    CUDA context and, under torchrun, NCCL threads holding locks.  Requests
    and results travel as length-prefixed pickles over the workers' pipes;
    one host thread per worker pulls the next chunk of the batch (longest
    queries first) as soon as its worker is free."""

    def __init__(self, workers: int) -> None:
        import subprocess
        import sys

        pkg_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        env = dict(os.environ)
        env["PYTHONPATH"] = pkg_root + os.pathsep + env.get("PYTHONPATH", "")
        import threading

        self._lock = threading.Lock()
        self.workers = workers
        self.procs = [subprocess.Popen([sys.executable, "-m", __package__ + ".compile_worker"],
                                       stdin=subprocess.PIPE, stdout=subprocess.PIPE, env=env)
                      for _ in range(workers)]
        # every worker answers one empty request before any timed use
        for p in self.procs:
            self._send(p, [])
        for p in self.procs:
            self._recv(p)

    @staticmethod
    def _send(proc, obj) -> None:
        import pickle
        import struct

        data = pickle.dumps(obj, protocol=pickle.HIGHEST_PROTOCOL)
        proc.stdin.write(struct.pack("<Q", len(data)) + data)
        proc.stdin.flush()

    @staticmethod
    def _recv(proc):
        import pickle
        import struct

        head = proc.stdout.read(8)
        if len(head) != 8:
            raise RuntimeError("compile worker exited")
        (n,) = struct.unpack("<Q", head)
        got = pickle.loads(proc.stdout.read(n))
        if isinstance(got, BaseException):
            raise got
        return got

    def compile(self, queries, on_chunk=None, light: bool = False
                ) -> List[Tuple[Optional[CompiledQuery], Optional[str]]]:
        """Compile a batch; ``on_chunk(indices, results)`` (optional) is
        called as each chunk of the batch completes, from a driver thread.
        Concurrent calls (the two-tier checker's overlap) take turns."""
        with self._lock:
            return self._compile(queries, on_chunk, light)

    def _compile(self, queries, on_chunk, light):
        import threading

        items = [_portable(q) + (light,) for q in queries]
        # longest first (cost ~ assertion count): the big queries start in the
        # first wave and the small ones fill the gaps, so the batch's critical
        # path is close to its largest query
        order = sorted(range(len(items)), key=lambda i: -len(items[i][0]))
        chunk = max(1, -(-len(items) // (self.workers * 4)))
        chunks = [order[k:k + chunk] for k in range(0, len(order), chunk)]
        out: List[Tuple[Optional[CompiledQuery], Optional[str]]] = [None] * len(items)  # type: ignore
        lock = threading.Lock()
        errors: List[BaseException] = []

        def drive(proc) -> None:
            while True:
                with lock:
                    if not chunks or errors:
                        return
                    idxs = chunks.pop(0)
                try:
                    self._send(proc, [items[i] for i in idxs])
                    got = self._recv(proc)
                    for i, r in zip(idxs, got):
                        out[i] = r
                    if on_chunk is not None:
                        on_chunk(idxs, got)
                except BaseException as exc:  # surfaced to the caller below
                    with lock:
                        errors.append(exc)
                    return

        threads = [threading.Thread(target=drive, args=(p,)) for p in self.procs]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        return out

    def stream(self, jobs, on_done) -> None:
        """Serve compile jobs until a ``None`` job arrives: ``jobs`` is a
        queue.PriorityQueue of (priority, seq, index, item) -- item as for
        _compile_one -- and ``on_done(indices, results)`` is called per
        finished chunk (from a driver thread; it may enqueue more jobs).
        Blocks until every worker has drained; re-raises a worker failure."""
        import queue as _q
        import threading

        with self._lock:
            errors: List[BaseException] = []
            stop = threading.Event()

            def drive(proc) -> None:
                while not stop.is_set():
                    job = jobs.get()
                    if job[3] is None:
                        jobs.put(job)          # the sentinel stays for the others
                        return
                    # several jobs per round trip only while the queue is
                    # long and only for the same priority class: a full
                    # presolve (up to ~200 ms) sits on its site's critical
                    # path and is never queued behind another one
                    batch = [job]
                    while len(batch) < 4 and jobs.qsize() > 2 * len(self.procs):
                        try:
                            nxt = jobs.get_nowait()
                        except _q.Empty:
                            break
                        if nxt[3] is None or nxt[0] != job[0] or job[0] == 0:
                            jobs.put(nxt)
                            break
                        batch.append(nxt)
                    try:
                        self._send(proc, [b[3] for b in batch])
                        got = self._recv(proc)
                        on_done([b[2] for b in batch], got)
                    except BaseException as exc:  # surfaced to the caller below
                        errors.append(exc)
                        stop.set()
                        jobs.put((-1, -1, -1, None))
                        return

            threads = [threading.Thread(target=drive, args=(p,)) for p in self.procs]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
            if errors:
                raise errors[0]

    def close(self) -> None:
        for p in self.procs:
            try:
                p.stdin.close()
                p.wait(timeout=5)
            except Exception:
                p.kill()
        self.procs = []


def default_workers() -> int:
    """Host cores per GPU process (torchrun's LOCAL_WORLD_SIZE ranks share the
    host), one left for the process itself, at most 16."""
    n = os.cpu_count() or 1
    local = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
    return max(1, min(16, n // local - 1))


class SiteChecker:
    """Holds one device context; decides compiled queries in batches."""

    # batches at least this large are compiled on the worker pool
    POOL_MIN_BATCH = 8

    def __init__(self, device: int = 0, lib_path: Optional[str] = None,
                 limits: Optional[dict] = None, compile_workers: Optional[int] = None) -> None:
        self.engine = Engine(device, lib_path)
        self.limits = dict(DEFAULT_LIMITS)
        if limits:
            self.limits.update(limits)
        self.stats = BatchStats()
        # 0 / 1: compile inline; None: default_workers()
        self.compile_workers = default_workers() if compile_workers is None else compile_workers
        self._pool: Optional[CompilePool] = None
        # light first tier on the device before the full presolve
        self.two_tier = os.environ.get("MK_TWO_TIER", "1") != "0"
        # (t_ms, event, ...) records of the streaming pipeline when a list
        self.trace: Optional[list] = None
        import threading

        self._device_lock = threading.Lock()
        self._warm = False

    def close(self) -> None:
        if self._pool is not None:
            self._pool.close()
            self._pool = None
        self.engine.close()

    def compile(self, queries, light: bool = False
                ) -> List[Tuple[Optional[CompiledQuery], Optional[str]]]:
        if self.compile_workers > 1 and len(queries) >= self.POOL_MIN_BATCH:
            if self._pool is None:
                self._pool = CompilePool(self.compile_workers)
            return self._pool.compile(queries, light=light)
        return compile_all(queries, light)

    def pack(self, compiled: Sequence[Optional[CompiledQuery]]) -> Tuple[PackedSet, List[int]]:
        problems, offsets = [], []
        for cq in compiled:
            offsets.append(len(problems))
            if cq is not None:
                problems.extend(cq.problems)
        return PackedSet(problems), offsets

    def decide(self, compiled: Sequence[Tuple[Optional[CompiledQuery], Optional[str]]],
               packed: Optional[PackedSet] = None, offsets: Optional[List[int]] = None,
               budget_s: Optional[float] = None) -> List[QueryResult]:
        cqs = [c for c, _ in compiled]
        if packed is None:
            packed, offsets = self.pack(cqs)
        t0 = time.perf_counter()
        # the reference grants every query its own timeout (engine/state.py:38);
        # a batch gets the sum, capped; ``budget_s``: an absolute budget for
        # the batch (the first tier)
        lim = dict(self.limits)
        lim["max_seconds"] = (budget_s if budget_s is not None else
                              min(self.limits["max_seconds"] * max(len(compiled), 1), 3600.0))
        if budget_s is not None:
            lim.update(self.TIER1_LIMITS)
        with self._device_lock:   # one engine call at a time per context
            if budget_s is not None and not self._warm and packed.problems:
                # the first engine call of a context allocates its work
                # buffers (GiBs of box stacks); a short first-tier budget
                # must not pay for that: one untimed call first
                self.engine.solve_packed(packed, lim)
            if packed.problems:
                self._warm = True
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

    # first tier: device budget for the whole light batch (seconds): per query,
    # clamped.  Measured on the B200 (profiles/r02_e2e_tiers_budget.jsonl):
    # config3 end to end is within noise for 5, 10 and 20 ms caps (the compile
    # pool is the critical path) and the 10 ms cap keeps the device step short
    TIER1_S = (0.0005, 0.002, 0.01)   # per query, minimum, maximum
    # smaller calls (analyze()'s one query per site) skip the first tier: a
    # query the light tier leaves undecided is compiled twice, which only
    # pays off amortised over a batch (measured on the B200, analyze() with
    # device screening: rms_norm 79 -> 50 ms, silu_and_mul 38 -> 18 ms,
    # paged_attention_v1 473 -> 414 ms; profiles/r02_analyze_tiers.jsonl)
    TWO_TIER_MIN = 8
    # extra engine limits of a first-tier call: no adaptive probe (a short
    # budgeted call gains nothing from the probe's restart; measured on the
    # B200: config3's first-tier device time 86 -> 72 ms per check_queries
    # call, profiles/r02_e2e_tiers_probe.jsonl) and split arity 8: on the
    # light problems a 10 ms budget leaves 60 undecided at 8, 78 at the full
    # problems' 12 (profiles/r02_tier1_split_k.jsonl)
    TIER1_LIMITS: Dict[str, object] = {"chunk": 65536, "split_k": 8}

    def tier1_budget(self, n: int) -> float:
        per, lo, hi = self.TIER1_S
        return min(max(per * n, lo), hi)

    def check_queries(self, queries: Sequence[Tuple[Sequence[ir.Node], Callable[[str], str]]]
                      ) -> List[QueryResult]:
        """Two tiers.  (1) Every query compiled *light* (structural presolve
        only) and searched on the device within a short budget: whatever the
        device decides (sat with its canonical witness, or unsat) is final --
        the model set and the witness order are the same as after the full
        presolve.  (2) The rest -- queries the light compile cannot bound or
        the budget did not finish -- through the full presolve and the
        device with the reference's per-query budget.  ``two_tier = False``
        runs (2) alone."""
        if not self.two_tier or len(queries) < self.TWO_TIER_MIN:
            return self._check_full(queries)
        if self.compile_workers > 1 and len(queries) >= self.POOL_MIN_BATCH:
            # the caller's process unpickles every compiled query the pool
            # returns; a cyclic-GC pass over a large heap in the middle of
            # that measured 45-55 ms per call (the results are acyclic, so
            # reference counting frees them; collection resumes afterwards)
            import gc

            was = gc.isenabled()
            gc.disable()
            try:
                return self._check_streaming(queries)
            finally:
                if was:
                    gc.enable()
        light = compile_all(queries, light=True)
        ok = [i for i, (cq, _) in enumerate(light) if cq is not None]
        out: List[Optional[QueryResult]] = [None] * len(queries)
        if ok:
            res = self.decide([light[i] for i in ok], budget_s=self.tier1_budget(len(ok)))
            for i, r in zip(ok, res):
                if r.status in ("sat", "unsat"):
                    out[i] = r
                    self.stats.tier1_decided += 1
        redo = [i for i, r in enumerate(out) if r is None]
        if redo:
            for i, r in zip(redo, self._check_full([queries[i] for i in redo])):
                out[i] = r
        self.stats.tier2_queries += len(redo)
        return out  # type: ignore[return-value]

    def _check_streaming(self, queries) -> List[QueryResult]:
        """The two tiers as one stream over the worker pool and the device:
        light compiles flow to the device's first tier as they finish; a
        query the light compile cannot bound, or the first tier does not
        decide, goes back to the pool for its full presolve (ahead of the
        remaining light compiles) and then to the device's second tier.  The
        device thread decides whatever has arrived in one batch per tier."""
        import itertools
        import queue
        import threading

        if self._pool is None:
            self._pool = CompilePool(self.compile_workers)
        n = len(queries)
        items = [_portable(q) for q in queries]
        jobs: "queue.PriorityQueue" = queue.PriorityQueue()
        seq = itertools.count()
        for i in sorted(range(n), key=lambda i: -len(items[i][0])):
            jobs.put((1, next(seq), i, items[i] + (True,)))       # light first
        ready: "queue.Queue" = queue.Queue()
        out: List[Optional[QueryResult]] = [None] * n
        failure: List[BaseException] = []

        t00 = time.perf_counter()
        trace = self.trace

        def ev(*what) -> None:
            if trace is not None:
                trace.append((round((time.perf_counter() - t00) * 1e3, 2),) + what)

        def on_done(idxs, results) -> None:
            ev("compiled", list(idxs))
            for i, r in zip(idxs, results):
                ready.put((i, r))

        def full_job(i) -> None:
            jobs.put((0, next(seq), i, items[i] + (False,)))      # ahead of light jobs

        def device_loop() -> None:
            done = 0
            light_seen = set()
            while done < n and not failure:
                batch = [ready.get()]
                while True:
                    try:
                        batch.append(ready.get_nowait())
                    except queue.Empty:
                        break
                if any(b is None for b in batch):
                    return
                tier1, tier2 = [], []
                for i, (cq, err) in batch:
                    if i not in light_seen:
                        light_seen.add(i)
                        if cq is None:
                            full_job(i)            # the light compile cannot bound it
                        else:
                            tier1.append((i, (cq, err)))
                    else:
                        tier2.append((i, (cq, err)))
                try:
                    if tier1:
                        ev("tier1", [i for i, _ in tier1])
                        t1 = time.perf_counter()
                        res = self.decide([c for _, c in tier1],
                                          budget_s=self.tier1_budget(len(tier1)))
                        self.stats.tier1_batches += 1
                        self.stats.tier1_s += time.perf_counter() - t1
                        for (i, _), r in zip(tier1, res):
                            if r.status in ("sat", "unsat"):
                                out[i] = r
                                done += 1
                                self.stats.tier1_decided += 1
                            else:
                                full_job(i)
                    if tier2:
                        ev("tier2", [i for i, _ in tier2])
                        t2 = time.perf_counter()
                        res = self.decide([c for _, c in tier2])
                        self.stats.tier2_batches += 1
                        self.stats.tier2_s += time.perf_counter() - t2
                        for (i, _), r in zip(tier2, res):
                            out[i] = r
                            done += 1
                            self.stats.tier2_queries += 1
                except BaseException as exc:  # surfaced to the caller below
                    failure.append(exc)
                ev("device_idle", done)
            jobs.put((2, next(seq), -1, None))                     # stop the pool

        th = threading.Thread(target=device_loop)
        th.start()
        t0 = time.perf_counter()
        try:
            self._pool.stream(jobs, on_done)
        except BaseException as exc:
            failure.append(exc)
            ready.put(None)
        finally:
            self.stats.compile_s += time.perf_counter() - t0
            th.join()
        if failure:
            raise failure[0]
        return out  # type: ignore[return-value]

    def _check_full(self, queries) -> List[QueryResult]:
        if self.compile_workers > 1 and len(queries) >= self.POOL_MIN_BATCH:
            return self._check_pipelined(queries)
        t0 = time.perf_counter()
        compiled = self.compile(queries)
        self.stats.compile_s += time.perf_counter() - t0
        return self.decide(compiled)

    def _check_pipelined(self, queries) -> List[QueryResult]:
        """Compile on the worker pool and decide on the device at the same
        time: compiled chunks (longest queries first) go to a device thread
        that decides whatever has arrived in one batch while the rest still
        compiles (the engine call releases the GIL).  Results are the same
        as compile-then-decide: queries are independent."""
        import queue
        import threading

        if self._pool is None:
            self._pool = CompilePool(self.compile_workers)
        arrivals: "queue.Queue" = queue.Queue()
        out: List[Optional[QueryResult]] = [None] * len(queries)
        failure: List[BaseException] = []

        def device_loop() -> None:
            while True:
                batch = [arrivals.get()]
                while True:
                    try:
                        batch.append(arrivals.get_nowait())
                    except queue.Empty:
                        break
                stop = any(b is None for b in batch)
                flat = [pair for chunk in batch if chunk is not None for pair in chunk]
                if flat and not failure:
                    try:
                        res = self.decide([r for _, r in flat])
                        for (i, _), rr in zip(flat, res):
                            out[i] = rr
                    except BaseException as exc:  # surfaced to the caller below
                        failure.append(exc)
                if stop:
                    return

        th = threading.Thread(target=device_loop)
        th.start()
        t0 = time.perf_counter()
        try:
            self._pool.compile(queries, on_chunk=lambda idxs, rs: arrivals.put(list(zip(idxs, rs))))
        finally:
            self.stats.compile_s += time.perf_counter() - t0
            arrivals.put(None)
            th.join()
        if failure:
            raise failure[0]
        return out  # type: ignore[return-value]

    def check(self, assertions: Sequence[ir.Node], origin_of: Callable[[str], str]) -> QueryResult:
        return self.check_queries([(assertions, origin_of)])[0]

    def feasible(self, assertions: Sequence[ir.Node], origin_of: Callable[[str], str],
                 max_seconds: Optional[float] = None) -> QueryResult:
        """Verdict only (sat / unsat / unknown), the reference's
        ``Solver.check(...).status`` (solver/interface.py:49-86): the engine
        stops at the first model (MK_PF_ANY) instead of the canonical one.
        ``reason`` is "budget" when the device search ran out of time (the
        query itself is decidable), else the compiler's give-up reason."""
        t0 = time.perf_counter()
        compiled = self.compile([(assertions, origin_of)])
        self.stats.compile_s += time.perf_counter() - t0
        cq = compiled[0][0]
        if cq is not None:
            for p in cq.problems:
                p.any_model = True
        saved = dict(self.limits)
        if max_seconds is not None:
            self.limits["max_seconds"] = max_seconds
        try:
            res = self.decide(compiled)[0]
        finally:
            self.limits = saved
        if res.status == "unknown" and cq is not None and res.reason is None \
                and not any(g.status == "unknown" for g in cq.groups):
            res.reason = "budget"
        return res
