"""BE-RRT# batch driver (Alg. 3) over a pre-generated RRG.

Harness code above the C ABI: it replays the exploration phase (the
generator's batches) into any context exposing
``append(h_new, src, dst, cost, flags=...) -> n_new_promising`` and
``exploit() -> stats`` and applies the Alg. 3 guard ``if |B'| > |B|: Replan``
 in its R10 form (``n_new_promising > 0``), followed by one
final unconditional exploit.  S = 1 is PI-RRT# (Alg. 1); S = N
is the PRM*-like single solve.
"""
from __future__ import annotations

from typing import Callable, Iterable, Optional

EDGES_UNDIRECTED = 4


def batches(n: int, S: int, start: int = 2) -> Iterable[tuple[int, int]]:
    """[a, b) vertex-id ranges of size S covering [start, n) (last one ragged)."""
    a = start
    while a < n:
        b = min(n, a + S)
        yield a, b
        a = b


def replay(ctx, graph, S: int, n_stop: Optional[int] = None, undirected: bool = True,
           on_exploit: Optional[Callable] = None, final: bool = True, start: int = 2):
    """Run Alg. 3 on ``ctx`` over vertices [start, n_stop) of ``graph``.

    ``on_exploit(k, a, b, stats)`` is called after every exploit.  Returns the
    list of (a, b, n_new_promising, stats-or-None) per batch."""
    n_stop = graph.n if n_stop is None else n_stop
    log = []
    for k, (a, b) in enumerate(batches(n_stop, S, start)):
        src, dst, cost = graph.batch(a, b, directed=not undirected)
        nprom = ctx.append(graph.h[a:b], src, dst, cost,
                           flags=EDGES_UNDIRECTED if undirected else 0)
        st = None
        if nprom > 0:                       # Alg. 3 line 10: |B'| > |B|
            st = ctx.exploit()
            if on_exploit:
                on_exploit(k, a, b, st)
        log.append((a, b, nprom, st))
    if final:                               # final unconditional replan
        st = ctx.exploit()
        if on_exploit:
            on_exploit(-1, n_stop, n_stop, st)
        log.append((n_stop, n_stop, 0, st))
    return log
