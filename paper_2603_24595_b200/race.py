"""K2 host side: build the race-sweep program of one store site at one
concrete launch (include/mk_b200.h mk_race_sweep).

The reference's race query for a store (engine/detectors.py:204-232) is

    path(t) + path(t') + [off(t) == off(t')] + [distinct(t, t')]

with every thread-private symbol (engine/state.py:32: thread ids, loop
indices, havoc loads) primed in the twin.  Fixing every other symbol (the
launch: BS/SL/TC, scalar arguments, launch dimensions, tensor fields) to the
values of a concrete launch leaves one thread's path over its private
symbols.  ``race_program`` compiles that path and the byte offset into a
narrow bytecode problem over the instance box; the device enumerates every
instance, sorts (offset, block) keys and scans for conflicts.

Loop-exit symbols of a thread-partitioned loop summary
(engine/executor.py:695-712: ``e >= init``, ``!(e < bound)``,
``(e - init) emod step == 0``) that appear nowhere else are pinned to the
concrete exit value (the least such ``e``): a value exists iff the least one
does, so the sweep's answer is unchanged and the instance box stays finite.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Mapping, Optional, Sequence, Tuple

from . import ir
from .compiler import (CompileError, Problem, _Emitter, _Ivl, _Lin, _Presolve, _may_err,
                       _truth, linear_truth, narrow_proof)

THREAD_PRIVATE = frozenset({"thread-id", "loop-index", "havoc"})   # engine/state.py:32
ID_NAMES = ("blockIdx.x", "blockIdx.y", "blockIdx.z", "threadIdx.x", "threadIdx.y", "threadIdx.z")
MAX_INSTANCES = (1 << 31) - 1
MAX_INNER = 1 << 16          # existential points tried per instance


class NotSweepable(Exception):
    """The store's instance box at this launch is not finite / too large /
    not provably narrow."""


@dataclass
class RaceProgram:
    problem: Problem
    off_reg: int
    shared: bool
    id_var: List[int]                       # ID_NAMES order, -1 when fixed / absent
    fixed: Dict[str, int] = field(default_factory=dict)   # pinned private symbols
    path: List[ir.Node] = field(default_factory=list)     # substituted path atoms
    offset: Optional[ir.Node] = None                      # substituted byte offset
    defs: Dict[str, ir.Node] = field(default_factory=dict)  # lattice-eliminated symbols
    n_exist: int = 0                                      # trailing existential vars

    @property
    def n_lead(self) -> int:
        return self.problem.nvars - self.n_exist

    @property
    def instances(self) -> int:
        """Instances of the leading vars (one access each at most)."""
        p, v = self.problem, 1
        for a, b in zip(p.lo[:self.n_lead], p.hi[:self.n_lead]):
            v *= b - a + 1
        return v

    @property
    def inner(self) -> int:
        p, v = self.problem, 1
        for a, b in zip(p.lo[self.n_lead:], p.hi[self.n_lead:]):
            v *= b - a + 1
        return v

    def decode(self, idx: int, nvars: Optional[int] = None) -> Dict[str, int]:
        """Index -> symbol values of the first ``nvars`` vars (default: the
        leading ones) in the device's order: last symbol fastest, every
        symbol ascending."""
        p = self.problem
        nv = self.n_lead if nvars is None else nvars
        vals = [0] * nv
        for i in range(nv - 1, -1, -1):
            s = p.hi[i] - p.lo[i] + 1
            vals[i] = p.lo[i] + idx % s
            idx //= s
        out = dict(self.fixed)
        out.update(zip(p.var_names[:nv], vals))
        for n, e in self.defs.items():
            if set(ir.symbols_of(e)) <= set(out):
                out[n] = ir.evaluate(e, out)
        return out


def split_race_query(assertions: Sequence[ir.Node]) -> Tuple[List[ir.Node], ir.Node, bool]:
    """(path(t), off(t), shared) of a recorded store-site race query."""
    if len(assertions) < 2 or (len(assertions) - 2) % 2:
        raise NotSweepable("not a race query")
    n = (len(assertions) - 2) // 2
    eq, dist = assertions[-2], assertions[-1]
    if eq[0] != "p" or eq[1] != "eq":
        raise NotSweepable("no offset equality")
    shared = dist[0] == "o" and dist[1] == "and"
    return list(assertions[:n]), eq[2], shared


def _exit_value(e: str, atoms: Sequence[ir.Node]) -> Optional[Tuple[ir.Node, List[int]]]:
    """Concrete exit value of a summarised loop's exit symbol ``e`` when its
    only atoms are the summary's three (returns the value and their indices)."""
    mine = [i for i, a in enumerate(atoms) if e in ir.symbols_of(a)]
    if len(mine) != 3:
        return None
    init = bound = step = None
    for i in mine:
        a = atoms[i]
        if a[0] == "p" and a[1] == "ge" and a[2][0] == "s" and a[2][1] == e:
            init = a[3]
        elif a[0] == "o" and a[1] == "not" and a[2][0][0] == "p" and a[2][0][1] == "lt" \
                and a[2][0][2][0] == "s" and a[2][0][2][1] == e and a[2][0][3][0] == "c":
            bound = a[2][0][3][1]
        elif a[0] == "p" and a[1] == "eq" and a[3][0] == "c" and a[3][1] == 0 \
                and a[2][0] == "b" and a[2][1] == "emod" and a[2][3][0] == "c":
            step = a[2][3][1]
    if init is None or bound is None or not step or step < 0:
        return None
    w = "i64"
    init64 = ("x", init, w)
    ceil_q = ("b", "div", ("b", "add", ("b", "sub", ("c", bound, w), init64, w),
                           ("c", step - 1, w), w), ("c", step, w), w)
    value = ("i", ("p", "ge", init64, ("c", bound, w)), init64,
             ("b", "add", init64, ("b", "mul", ("c", step, w), ceil_q, w), w), w)
    return value, mine


class _BoundsOnly(_Presolve):
    """The compiler's presolve restricted to sound bound propagation and
    lattice substitution (a loop index ``i = init + step*k`` is enumerated
    through ``k``): no order-driven elimination or aggregation, so every
    thread identity symbol stays an enumerated coordinate; fixed symbols are
    recorded."""

    def __init__(self, *a, **kw) -> None:
        super().__init__(*a, **kw)
        self.fixed: Dict[str, int] = {}

    def _substitute_many(self, m):
        for name, e in m.items():
            if e[0] == "c":
                self.fixed[name] = e[1]
        super()._substitute_many(m)

    def _try_eliminate(self, lin):
        return False

    def _try_aggregate(self, lin):
        return False

    def _try_aggregate_ineq(self, lin):
        return False


def _components(atoms: Sequence[ir.Node]) -> List[Tuple[set, List[int]]]:
    parent: Dict[str, str] = {}

    def find(x: str) -> str:
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    syms = [set(ir.symbols_of(a)) for a in atoms]
    for vs in syms:
        for v in vs:
            parent.setdefault(v, v)
        vs = list(vs)
        for o in vs[1:]:
            ra, rb = find(vs[0]), find(o)
            if ra != rb:
                parent[ra] = rb
    groups: Dict[str, Tuple[set, List[int]]] = {}
    for i, vs in enumerate(syms):
        if not vs:
            continue
        r = find(next(iter(vs)))
        g = groups.setdefault(r, (set(), []))
        g[0].update(vs)
        g[1].append(i)
    return list(groups.values())


def _box_satisfiable(atoms: Sequence[ir.Node], names: Sequence[str],
                     bounds: Mapping[str, Tuple[int, int]], limit: int = 1 << 22) -> bool:
    vol = 1
    for n in names:
        vol *= bounds[n][1] - bounds[n][0] + 1
    if vol > limit:
        raise NotSweepable(f"side component of {vol} points")
    for idx in range(vol):
        x = {}
        for n in reversed(names):
            lo, hi = bounds[n]
            s = hi - lo + 1
            x[n] = lo + idx % s
            idx //= s
        if all(_truthy(a, x) for a in atoms):
            return True
    return False


def race_program(assertions: Sequence[ir.Node], origin_of: Callable[[str], str],
                 launch: Mapping[str, int], max_instances: int = MAX_INSTANCES) -> RaceProgram:
    """The sweep program of a store-site race query at a concrete launch
    (``launch`` must give a value to every non-private symbol; a finding's
    witness does)."""
    path, off, shared = split_race_query(assertions)
    return path_program(path, off, shared, origin_of, launch, max_instances)


def path_program(path: Sequence[ir.Node], off: ir.Node, shared: bool,
                 origin_of: Callable[[str], str], launch: Mapping[str, int],
                 max_instances: int = MAX_INSTANCES,
                 id_extents: Optional[Mapping[str, int]] = None) -> RaceProgram:
    """One thread's access program (path atoms, byte offset) at a concrete
    launch.  With ``id_extents`` (thread-id name -> launch extent) every id
    of extent > 1 is an enumerated coordinate even when the path and offset
    never mention it (the concrete oracle runs every thread of the launch,
    SPEC.md:586-600); without it only the mentioned ids are, as the
    reference's symbolic twin query has them (engine/detectors.py:234-273)."""
    names: Dict[str, str] = {}
    for a in path:
        ir.symbols_of(a, names)
    ir.symbols_of(off, names)
    private = {n: w for n, w in names.items() if origin_of(n) in THREAD_PRIVATE}
    outer = [n for n in names if n not in private]
    missing = [n for n in outer if n not in launch]
    if missing:
        raise NotSweepable(f"launch does not fix {missing[:4]}")
    if any(ir.is_float(w) for w in private.values()):
        raise NotSweepable("float private symbol")
    sub = {n: ("c", int(launch[n]), names[n]) for n in outer}
    atoms = [ir.simplify(ir.substitute(a, sub)) for a in path]
    offset = ir.simplify(ir.substitute(off, sub))
    atoms = [a for a in atoms if a != ir.TRUE]
    if any(a == ir.FALSE for a in atoms):
        raise NotSweepable("path infeasible at this launch")
    if any(_has_float_node(a) for a in atoms) or _has_float_node(offset):
        raise NotSweepable("float atoms")
    # concrete exit values of summarised loops
    off_syms = set(ir.symbols_of(offset))
    exits: Dict[str, ir.Node] = {}
    for n in sorted(private):
        if origin_of(n) == "loop-index" and ".exit$" in n and n not in off_syms \
                and n not in ID_NAMES:
            got = _exit_value(n, atoms)
            if got is not None:
                exits[n] = got[0]
    if exits:
        # the pinned value satisfies its own three summary atoms by
        # construction (>= init, >= bound, congruent to init): drop them
        summary = set()
        for n in exits:
            summary.update(_exit_value(n, atoms)[1])
        atoms = [a for i, a in enumerate(atoms) if i not in summary]
        atoms = [ir.simplify(ir.substitute(a, exits)) for a in atoms]
        atoms = [a for a in atoms if a != ir.TRUE]
    # sound bounds (and lattice coordinates) of the remaining private symbols
    widths = {n: w for n, w in private.items() if n not in exits}
    # thread identities first: a lattice substitution then always eliminates
    # the loop index, never an identity (compiler._Presolve._try_lattice)
    order = [n for n in ID_NAMES if n in widths] + sorted(n for n in widths if n not in ID_NAMES)
    ps = _BoundsOnly(list(atoms), dict(widths), {n: float(i) for i, n in enumerate(order)},
                     {n: False for n in widths})
    try:
        ps.run()
    except CompileError as exc:
        raise NotSweepable(str(exc))
    if ps.unsat:
        raise NotSweepable("path infeasible at this launch")
    fixed = dict(ps.fixed)
    defs = {n: e for n, e in ps.defs.items() if n not in fixed}
    if any(n in defs for n in ID_NAMES):
        raise NotSweepable("thread identity eliminated by presolve")
    # exact atoms over the enumerated coordinates: fixed values and lattice
    # definitions substituted into the original atoms and the offset
    rewrite = {n: ("c", v, widths.get(n, "i64")) for n, v in fixed.items()}
    rewrite.update(defs)
    atoms = [ir.simplify(ir.substitute(a, rewrite)) for a in atoms]
    atoms = [a for a in atoms if a != ir.TRUE]
    if any(a == ir.FALSE for a in atoms):
        raise NotSweepable("path infeasible at this launch")
    offset = ir.simplify(ir.substitute(offset, rewrite))
    atoms = [a for a in atoms if not _lattice_tautology(a)]
    bounds: Dict[str, Tuple[int, int]] = {}
    free = set()
    for a in atoms:
        free |= set(ir.symbols_of(a))
    free |= set(ir.symbols_of(offset))
    free |= {n for n in ID_NAMES if n in widths and n not in fixed}
    extra: Dict[str, Tuple[int, int]] = {}
    if id_extents:
        for n in ID_NAMES:
            if n not in widths and n not in fixed and id_extents.get(n, 1) > 1:
                extra[n] = (0, int(id_extents[n]) - 1)
        free |= set(extra)
    for n in free:
        if n in extra:
            bounds[n] = extra[n]
            continue
        b = ps.bounds.get(n)
        if b is None:
            b = ir.bounds(widths[n]) if n in widths else (None, None)
        if b[0] is None or b[1] is None:
            raise NotSweepable(f"{n} unbounded")
        bounds[n] = b
    # atoms that hold without error on the whole box (sound interval proof)
    ivl = _Ivl(dict(bounds))
    atoms = [a for a in atoms
             if _may_err(a) or (_truth(a, ivl) != "T" and linear_truth(a, ivl) != "T")]
    # components touching neither the offset nor a thread identity only
    # gate feasibility: decide them once and drop them
    relevant = set(ir.symbols_of(offset)) | {n for n in ID_NAMES if n in free}
    keep: List[ir.Node] = []
    for vs, idxs in _components(atoms):
        comp = [atoms[i] for i in idxs]
        if vs & relevant:
            keep.extend(comp)
        elif not _box_satisfiable(comp, sorted(vs), bounds):
            raise NotSweepable("path infeasible at this launch")
    keep.extend(a for a in atoms if not ir.symbols_of(a))
    atoms = keep
    # leading vars: the instance (offset / identity symbols); trailing vars
    # are existential (an instance is one access iff some value works)
    lead = sorted(relevant)
    exist = sorted({n for a in atoms for n in ir.symbols_of(a)} - relevant)
    var_names = lead + exist
    lo = [bounds[n][0] for n in var_names]
    hi = [bounds[n][1] for n in var_names]
    vol = 1
    for a, b in zip(lo[:len(lead)], hi[:len(lead)]):
        vol *= b - a + 1
    if vol > max_instances:
        raise NotSweepable(f"{vol} instances")
    if len(var_names) > 8:
        raise NotSweepable(f"{len(var_names)} private symbols (> 8)")
    inner = 1
    for a, b in zip(lo[len(lead):], hi[len(lead):]):
        inner *= b - a + 1
    if inner > MAX_INNER:
        raise NotSweepable(f"{inner} existential points per instance")
    index = {n: i for i, n in enumerate(var_names)}
    em = _Emitter(index)
    for i, a in enumerate(atoms):
        em.atom(a, i)
    r_off = em.emit(offset)
    code, nregs, regs = em.finish([r_off])
    masks = []
    for a in atoms:
        m = 0
        for n in ir.symbols_of(a):
            m |= 1 << index[n]
        masks.append(m)
    prob = Problem(var_names=var_names, lo=lo, hi=hi, maximize=[False] * len(var_names),
                   insns=code, consts=list(em.consts), nregs=max(nregs, 1),
                   atom_regs=[0] * len(atoms), atom_masks=masks, rows=[],
                   ops_per_point=len(code))
    prob.narrow = narrow_proof(prob)
    if not prob.narrow:
        raise NotSweepable("not provably narrow")
    id_var = [index.get(n, -1) for n in ID_NAMES]
    return RaceProgram(problem=prob, off_reg=regs[0], shared=shared, id_var=id_var,
                       n_exist=len(exist),
                       fixed={n: v for n, v in fixed.items() if n in ID_NAMES or n in private},
                       path=list(atoms), offset=offset, defs=defs)


def _lattice_tautology(a: ir.Node) -> bool:
    """``emod(L, m) == 0`` with L linear and every coefficient and the
    constant divisible by m: true at every point (the loop-summary congruence
    after its lattice substitution, engine/executor.py:680-684)."""
    if not (a[0] == "p" and a[1] == "eq" and a[3][0] == "c" and a[3][1] == 0):
        return False
    e = a[2]
    if not (e[0] == "b" and e[1] == "emod" and e[3][0] == "c" and e[3][1] != 0):
        return False
    m = abs(e[3][1])
    try:
        terms, c0 = _Lin({}).lin(e[2])
    except Exception:
        return False
    if any(not isinstance(k, str) for k in terms):
        return False
    return c0 % m == 0 and all(v % m == 0 for v in terms.values())


def _has_float_node(e: ir.Node) -> bool:
    t = e[0]
    if t in ("c", "s"):
        return ir.is_float(e[2])
    if t in ("b", "x", "i") and ir.is_float(e[-1]):
        return True
    return any(_has_float_node(c) for c in ir.children(e))


def brute_force(prog: RaceProgram) -> Tuple[int, int, bool]:
    """Pure-Python restatement of the sweep for small launches (tests only):
    (tuples, conflicting adjacent pairs in (key, index) order, has_race)."""
    tuples = []
    nv = prog.problem.nvars
    for idx in range(prog.instances):
        for j in range(prog.inner):
            x = prog.decode(idx * prog.inner + j, nv)
            if all(_truthy(a, x) for a in prog.path):
                off = ir.evaluate(prog.offset, x)
                blk = tuple(x.get(n, 0) for n in ID_NAMES[:3]) if prog.shared else ()
                tuples.append(((off, blk), idx, x))
                break
    tuples.sort(key=lambda t: (t[0], t[1]))
    conflicts = 0
    for (k1, _, x1), (k2, _, x2) in zip(tuples, tuples[1:]):
        if k1 != k2:
            continue
        ids = ID_NAMES[3:] if prog.shared else ID_NAMES
        if any(x1.get(n, 0) != x2.get(n, 0) for n in ids):
            conflicts += 1
    # existence does not depend on the order inside a segment
    by_key: Dict[Tuple, set] = {}
    for k, _, x in tuples:
        ids = ID_NAMES[3:] if prog.shared else ID_NAMES
        by_key.setdefault(k, set()).add(tuple(x.get(n, 0) for n in ids))
    has = any(len(v) > 1 for v in by_key.values())
    return len(tuples), conflicts, has


def _truthy(a: ir.Node, x: Mapping[str, int]) -> bool:
    try:
        return bool(ir.evaluate(a, x))
    except ir.EvalError:
        return False
