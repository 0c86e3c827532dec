"""Witness replay (SPEC.md:573-631 ``replay_witness``; the reference does not
ship its oracle): confirm a sat finding's canonical witness in two ways.

* **Expression level** -- the witness satisfies every assertion of the
  site query in mathematical mode (``solver/query.py:45-62``, the same
  predicate the reference validates models with): the violated bound of an
  overflow / out-of-bounds site is reproduced by direct evaluation.
* **Full launch** -- every launch-level symbol (BS, SL, TC, launch
  dimensions, scalar arguments, tensor extents) is fixed to the witness and
  *every thread of that launch* is checked on the B200: the site query
  becomes a per-thread program over all block and thread ids (loop indices
  and loaded values existential), swept by the K2 machinery
  (``race.path_program`` -> ``mk_race_sweep``).  The sweep counts the
  threads that violate the site at the witness launch; the finding is
  confirmed when the witness is a model and at least one thread violates
  (the witness's own thread is one of them).

A witness whose launch does not fit the sweep (more than 2^31 - 1 thread
instances, float private symbols) is confirmed at expression level only, as
SPEC.md allows for witnesses that exceed the concrete cap.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, Mapping, Optional, Sequence

from . import ir, race

_DIMS = {"blockIdx.x": "gridDim.x", "blockIdx.y": "gridDim.y", "blockIdx.z": "gridDim.z",
         "threadIdx.x": "blockDim.x", "threadIdx.y": "blockDim.y", "threadIdx.z": "blockDim.z"}


@dataclass
class Replay:
    status: str                 # "confirmed" | "confirmed-expression" | "not-confirmed"
    expression: bool            # the witness satisfies every assertion
    full_launch: Optional[bool]  # None: launch not swept
    violating_threads: int = 0  # threads of the launch that violate the site
    candidates: int = 0         # threads enumerated: the launch's threads that bound
                                # propagation at the witness launch could not exclude
    note: str = ""


def launch_of(witness: Mapping[str, int], origin_of: Callable[[str], str]) -> Dict[str, int]:
    """Launch-level part of a witness: every symbol that is not thread
    private (engine/state.py:32)."""
    return {n: int(v) for n, v in witness.items()
            if "'" not in n and origin_of(n) not in race.THREAD_PRIVATE}


def replay_witness(engine, assertions: Sequence[ir.Node], origin_of: Callable[[str], str],
                   witness: Mapping[str, int],
                   max_instances: int = race.MAX_INSTANCES) -> Replay:
    expr = ir.is_model(assertions, witness)
    launch = launch_of(witness, origin_of)
    extents = {tid: int(launch[dim]) for tid, dim in _DIMS.items() if dim in launch}
    try:
        # the per-thread program: all assertions as the path, a constant
        # "offset" (the count of executing instances is what matters)
        prog = race.path_program(list(assertions), ("c", 0, "i64"), False, origin_of, launch,
                                 max_instances, id_extents=extents)
    except race.NotSweepable as exc:
        msg = str(exc)
        if "infeasible" in msg:
            return Replay("not-confirmed", expr, False, note=msg)
        return Replay("confirmed-expression" if expr else "not-confirmed", expr, None, note=msg)
    res = engine.race_sweep(prog)
    full = res["tuples"] > 0
    status = "confirmed" if (expr and full) else "not-confirmed"
    return Replay(status, expr, full, int(res["tuples"]), int(res["instances"]))
