"""Context inference: invocation log -> analysis
context, the domain the checking stage enumerates.

Restates ``minikernel.context.infer_context`` (context.py:315-395) and its
helpers ``_feature_names`` / ``_feature_value`` (:398-425), ``_classify``
(:427-440), ``_affine_fit`` (:443-466) and ``_check_soundness``
(:469-495), with the per-feature work done column-wise: every observed
feature of the kernel becomes one row of an integer matrix over the runs,
and each law (invariant, exact affine fit against TC / SL / BS, bound) is
decided for all rows at once.  The result is the reference's own
``AnalysisContext`` (built from its dataclasses), so ``context_to_json``,
``to_engine_facts`` and ``analyze`` consume it unchanged; errors are the
reference's ``ContextError`` with the same messages.

Float-valued features (scalar epsilons) cannot be exact affine laws; they
go through the same invariant / bound rules on their Python values.
"""

from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

_BASES = ("TC", "SL", "BS")        # the reference's fit order (context.py:432)


def _ref():
    from minikernel import context as C
    return C


def feature_names(obs) -> List[str]:
    """context.py:398-405."""
    if obs.kind == "scalar":
        return ["value"]
    names = [f"dim{i}" for i in range(len(obs.shape))]
    names += ["numel", "itemsize"]
    if obs.int_min is not None:
        names += ["int_min", "int_max"]
    return names


def feature_value(obs, feature: str):
    """context.py:408-425."""
    if feature == "value":
        return obs.value
    if feature == "numel":
        n = 1
        for d in obs.shape:
            n *= d
        return n
    if feature == "itemsize":
        return obs.itemsize
    if feature == "int_min":
        return obs.int_min
    if feature == "int_max":
        return obs.int_max
    if feature.startswith("dim"):
        return obs.shape[int(feature[3:])]
    raise _ref().ContextError(f"unknown feature {feature!r}")


def _affine_fits(V: np.ndarray, x: np.ndarray) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Exact integer laws v = a*x + b (a != 0) for every row of V at once
    (context.py:443-466): the first pair of runs with distinct x fixes
    (a, b), every run must then agree.  Returns (ok, a, b) per row."""
    F = V.shape[0]
    ok = np.zeros(F, dtype=bool)
    a = np.zeros(F, dtype=object)
    b = np.zeros(F, dtype=object)
    n = x.shape[0]
    pair = None
    for i in range(n):
        for j in range(i + 1, n):
            if x[i] != x[j]:
                pair = (i, j)
                break
        if pair:
            break
    if pair is None or F == 0:
        return ok, a, b
    i, j = pair
    dx = int(x[j] - x[i])
    dv = V[:, j] - V[:, i]
    div = np.array([int(d) % dx == 0 for d in dv], dtype=bool)
    av = np.array([int(d) // dx for d in dv], dtype=object)
    bv = V[:, i] - av * int(x[i])
    pred = av[:, None] * x[None, :].astype(object) + bv[:, None]
    agree = np.all(pred == V, axis=1)
    ok = div & (av != 0) & agree
    return ok, av, bv


def infer_context(log, kernel: str):
    """context.py:315-395: classify every observed feature of ``kernel``
    across the log's runs."""
    C = _ref()
    rows = [(run.batch_size, run.seq_len, call) for run in log.runs for call in run.calls
            if call.kernel == kernel]
    if not rows:
        raise C.ContextError(f"kernel {kernel!r} does not appear in the log")
    runs_with = [run for run in log.runs if any(c.kernel == kernel for c in run.calls)]
    if len(runs_with) < 4:
        raise C.ContextError(
            f"insufficient variation: kernel {kernel!r} appears in "
            f"{len(runs_with)} run(s); need at least 4")
    if len({r.batch_size for r in runs_with}) < 2 \
            or len({r.seq_len for r in runs_with}) < 2:
        raise C.ContextError(
            "insufficient variation: need at least two distinct batch "
            "sizes and two distinct sequence lengths")

    nargs = len(rows[0][2].args)
    keys: List[str] = []
    values: List[list] = []
    arg_meta: List[Tuple[int, str, str]] = []
    for pos in range(nargs):
        first = rows[0][2].args[pos]
        dtype = first.dtype
        for _, _, call in rows:
            obs = call.args[pos]
            if obs.kind == "tensor" and obs.dtype != dtype:
                raise C.ContextError(f"inconsistent dtype for arg {pos} of {kernel!r}")
        arg_meta.append((pos, first.kind, dtype))
        for fname in feature_names(first):
            keys.append(f"arg{pos}.{fname}")
            values.append([feature_value(call.args[pos], fname) for _, _, call in rows])

    bases = {
        "TC": np.array([bs * sl for bs, sl, _ in rows], dtype=object),
        "SL": np.array([sl for _, sl, _ in rows], dtype=object),
        "BS": np.array([bs for bs, _, _ in rows], dtype=object),
    }
    # integer features as one object matrix (exact Python ints: numel of a
    # large tensor exceeds int64 products in the fit)
    integral = [all(isinstance(v, int) for v in vs) for vs in values]   # context.py:431
    int_idx = [k for k, f in enumerate(integral) if f]
    fits: Dict[str, Tuple[np.ndarray, np.ndarray, np.ndarray]] = {}
    if int_idx:
        V = np.array([values[k] for k in int_idx], dtype=object)
        for basis in _BASES:
            fits[basis] = _affine_fits(V, bases[basis])
    where = {k: r for r, k in enumerate(int_idx)}

    classified: Dict[str, object] = {}
    for k, key in enumerate(keys):
        vs = values[k]
        feature = key.split(".", 1)[1]
        if all(v == vs[0] for v in vs):
            classified[key] = C.Constraint(feature, "invariant", value=vs[0])
            continue
        law = None
        if integral[k]:
            r = where[k]
            for basis in _BASES:
                ok, a, b = fits[basis]
                if ok[r]:
                    law = C.Constraint(feature, "linear", basis=basis, coeff=int(a[r]),
                                       offset=int(b[r]))
                    break
        if law is None:
            if feature == "int_min":
                law = C.Constraint(feature, "lower_bound", bound=min(vs))
            else:
                law = C.Constraint(feature, "upper_bound", bound=max(vs))
        classified[key] = law

    # equal classes: identical value vectors (type-tagged), in first-member order
    groups: Dict[Tuple, List[str]] = {}
    for k, key in enumerate(keys):
        vec = tuple((isinstance(v, int), v) for v in values[k])
        groups.setdefault(vec, []).append(key)
    order = {key: k for k, key in enumerate(keys)}
    equal = tuple(tuple(m) for m in sorted(groups.values(), key=lambda m: order[m[0]])
                  if len(m) >= 2)

    args = []
    for pos, kind, dtype in arg_meta:
        prefix = f"arg{pos}."
        args.append(C.ArgContext(position=pos, kind=kind, dtype=dtype,
                                 constraints=tuple(classified[k] for k in keys
                                                   if k.startswith(prefix))))
    ctx = C.AnalysisContext(kernel=kernel, args=tuple(args), equal=equal)
    check_soundness(ctx, rows)
    return ctx


def check_soundness(ctx, rows: Sequence[Tuple[int, int, object]]) -> None:
    """context.py:469-495: every emitted law holds on every observation and
    every equality class is an equality."""
    C = _ref()
    values: Dict[str, list] = {}
    for arg in ctx.args:
        for c in arg.constraints:
            vs = [feature_value(call.args[arg.position], c.feature) for _, _, call in rows]
            values[f"arg{arg.position}.{c.feature}"] = vs
            for (bs, sl, _), v in zip(rows, vs):
                basis = {"TC": bs * sl, "SL": sl, "BS": bs}
                if c.law == "invariant" and v != c.value:
                    raise C.ContextError(f"unsound invariant for {c.feature}")
                if c.law == "linear" and v != c.coeff * basis[c.basis] + c.offset:
                    raise C.ContextError(f"unsound linear law for {c.feature}")
                if c.law == "upper_bound" and v > c.bound:
                    raise C.ContextError(f"unsound upper bound for {c.feature}")
                if c.law == "lower_bound" and v < c.bound:
                    raise C.ContextError(f"unsound lower bound for {c.feature}")
    for cls in ctx.equal:
        base = values[cls[0]]
        for member in cls[1:]:
            if values[member] != base:
                raise C.ContextError(f"unsound equality class {cls}")


def infer_context_json(log_text: str, kernel: str, source_name: str = "<log>") -> str:
    """Log text -> canonical context JSON (the reference's parse_log and
    context_to_json around this module's inference)."""
    C = _ref()
    return C.context_to_json(infer_context(C.parse_log(log_text, source_name), kernel))
