"""ORACLE — test infrastructure only.  Exhaustive single-agent route enumerator, the independent
checker SPEC.md:245-246 and acceptance criterion 3 name for A* optimality.

Enumerates every stage sequence S₀ → (l−1 distinct stages) satisfying CC2 (≤ 1 descent, and
transposing it yields an increasing sequence), every node choice per stage, times
each route with the same cost model (λ + bytes/β hops, compute_fwd on the way out, mirrored
backward with compute × bwd_ratio, interval constraints deferring entry to the interval end) and
returns the minimum e2e.  Written independently of paper_2502_19913_b200.scheduler.
"""

import itertools
import math


def _valid_cc2(seq):
    descents = [i for i in range(1, len(seq)) if seq[i] < seq[i - 1]]
    if not descents:
        return True
    if len(descents) > 1:
        return False
    i = descents[0]
    t = list(seq)
    t[i - 1], t[i] = t[i], t[i - 1]
    return all(t[j] < t[j + 1] for j in range(len(t) - 1))


def _defer(windows, t, dur):
    changed = True
    while changed:
        changed = False
        for a, b in windows:
            if t < b and a < t + dur:
                t, changed = b, True
    return t


def route_e2e(nodes, origin, fwd, bwd, comm, windows):
    t = _defer(windows.get(origin, []), 0.0, fwd[origin]) + fwd[origin]
    prev = origin
    for v in nodes[1:]:
        arr = t + comm[prev][v]
        t = _defer(windows.get(v, []), arr, fwd[v]) + fwd[v]
        prev = v
    t = t + (comm[prev][origin] if prev != origin else 0.0)
    prev = origin
    for v in reversed(nodes[1:]):
        arr = t + comm[prev][v]
        t = _defer(windows.get(v, []), arr, bwd[v]) + bwd[v]
        prev = v
    arr = t + (comm[prev][origin] if prev != origin else 0.0)
    return _defer(windows.get(origin, []), arr, bwd[origin]) + bwd[origin]


def best_route(origin, stage_nodes, l, fwd, bwd, comm, banned=(), windows=None):
    """(min e2e, node sequence) over all CC2-valid routes of exactly l stages."""
    windows = windows or {}
    s = len(stage_nodes)
    best = (math.inf, None)
    for rest in itertools.permutations(range(1, s), l - 1):
        seq = (0,) + rest
        if not _valid_cc2(seq):
            continue
        choices = [[v for v in stage_nodes[st] if v not in banned] for st in rest]
        for pick in itertools.product(*choices):
            nodes = (origin,) + pick
            e = route_e2e(nodes, origin, fwd, bwd, comm, windows)
            if e < best[0] - 1e-12:
                best = (e, nodes)
    return best
