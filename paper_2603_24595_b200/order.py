"""Canonical witness order.

Restates ``_optimization_order`` (minikernel/engine/report.py:177-203):

1. ``BS``, ``SL``, ``TC``                          minimized
2. scalar-argument symbols, code-point sorted       minimized
3. ``blockIdx.{x,y,z}``, ``blockIdx.{x,y,z}'``,
   ``threadIdx.{x,y,z}``, ``threadIdx.{x,y,z}'``    maximized
4. loop-index symbols (primes included), sorted     minimized
5. everything else, sorted                          minimized

``origin_of`` follows ``SymbolTable.origin_of`` (engine/state.py:68-70):
twin primes share the origin of the symbol they shadow.
"""

from __future__ import annotations

from typing import Callable, Iterable, List, Mapping, Tuple

AXES = ("x", "y", "z")
ORIGIN_SCALAR = "scalar-arg"   # engine/state.py:29
ORIGIN_LOOP = "loop-index"     # engine/state.py:26


class OriginLookup:
    """``origin_of`` over a recorded {symbol: origin} map (picklable, so a
    query can be compiled in a worker process)."""

    __slots__ = ("origins",)

    def __init__(self, origins: Mapping[str, str]) -> None:
        self.origins = dict(origins)

    def __call__(self, name: str) -> str:
        return self.origins.get(name.rstrip("'"), "unknown")


def origin_lookup(origins: Mapping[str, str]) -> Callable[[str], str]:
    return OriginLookup(origins)


def optimization_order(names: Iterable[str],
                       origin_of: Callable[[str], str]) -> List[Tuple[str, str]]:
    present = set(names)
    order: List[Tuple[str, str]] = []
    taken = set()

    def take(name: str, direction: str) -> None:
        if name in present and name not in taken:
            order.append((name, direction))
            taken.add(name)

    for name in ("BS", "SL", "TC"):
        take(name, "min")
    for name in sorted(n for n in present if origin_of(n) == ORIGIN_SCALAR):
        take(name, "min")
    for stem in ("blockIdx", "threadIdx"):
        for prime in ("", "'"):
            for a in AXES:
                take(f"{stem}.{a}{prime}", "max")
    for name in sorted(n for n in present if origin_of(n) == ORIGIN_LOOP):
        take(name, "min")
    for name in sorted(present - taken):
        take(name, "min")
    return order
