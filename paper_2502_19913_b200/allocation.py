"""Node-to-stage allocation (§3.2, Eq. 1 at PAPER.md:196-198).

* ``stage_sizes``   Eq. 1 stage sizes, exact in integers or an error naming the nearest feasible
                    node counts.
* ``cluster_nodes`` size-constrained genetic partition minimising the slowest intra-cluster
                    DP-sync transfer.
* ``order_stages``  exact closed-loop TSP over clusters (Held-Karp), lexicographically smallest
                    optimal tour, S₀ = the unique largest cluster.

On a B200 box every link is identical, so the GA and the TSP are degenerate (any partition and
order is optimal; ties break lexicographically) and B200 configs pass an explicit
``StageAssignment``.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .errors import ValidationError
from .topology import Topology, comm_matrix

_TIE_EPS = 1e-9


def _as_fraction(x) -> Fraction:
    if isinstance(x, Fraction):
        return x
    if isinstance(x, int):
        return Fraction(x)
    return Fraction(x).limit_denominator(10**6)


# ---------------------------------------------------------------------------------------
# Eq. 1
# ---------------------------------------------------------------------------------------
def stage_sizes(n_nodes: int, s: int, k) -> list[int]:
    """|S_i| = |S_0|·(1 − (s/(s−1))·(k/100)) for i ≥ 1, Σ|S_i| = n_nodes."""
    if s < 2:
        raise ValidationError(f"need at least 2 stages, got s={s}")
    kf = _as_fraction(k)
    if kf < 0 or kf >= Fraction(100 * (s - 1), s):
        raise ValidationError(f"skip percent k={float(kf):g} must satisfy 0 <= k < {100 * (s - 1) / s:g} for s={s}")
    ratio = 1 - Fraction(s, s - 1) * kf / 100  # |S_i| / |S_0|, in (0, 1]
    # |S_0| = t·q and |S_i| = t·p with ratio = p/q in lowest terms => n = t·(q + (s−1)·p)
    p, q = ratio.numerator, ratio.denominator
    step = q + (s - 1) * p
    if n_nodes % step:
        lo = (n_nodes // step) * step
        near = [v for v in (lo, lo + step) if v > 0]
        raise ValidationError(
            f"Eq. 1 has no integral solution for n={n_nodes}, s={s}, k={float(kf):g}; "
            f"nearest feasible node counts: {near}"
        )
    t = n_nodes // step
    return [t * q] + [t * p] * (s - 1)


# ---------------------------------------------------------------------------------------
# StageAssignment
# ---------------------------------------------------------------------------------------
@dataclass(frozen=True)
class StageAssignment:
    """``members[c]`` = node ids of cluster c; ``order[i]`` = cluster running pipeline stage i.

    ``order[0]`` is S₀.  Pipeline stage i holds model layers [i·δ, (i+1)·δ)."""

    s: int
    sizes: list[int]
    members: list[list[int]]
    order: list[int]

    def __post_init__(self):
        if len(self.sizes) != self.s or len(self.members) != self.s or len(self.order) != self.s:
            raise ValidationError("assignment: sizes/members/order must each have s entries")
        if sorted(self.order) != list(range(self.s)):
            raise ValidationError(f"assignment: order {self.order} is not a permutation of 0..{self.s - 1}")
        seen: set[int] = set()
        for c, (sz, mem) in enumerate(zip(self.sizes, self.members)):
            if len(mem) != sz:
                raise ValidationError(f"assignment: cluster {c} has {len(mem)} members, size says {sz}", row=c)
            if seen & set(mem):
                raise ValidationError(f"assignment: node(s) {sorted(seen & set(mem))} in more than one cluster")
            seen |= set(mem)
        if seen != set(range(len(seen))):
            raise ValidationError("assignment: members must partition nodes 0..n-1")

    @property
    def n(self) -> int:
        return sum(self.sizes)

    def stage_nodes(self, stage: int) -> list[int]:
        """Nodes running pipeline stage ``stage`` (sorted)."""
        return sorted(self.members[self.order[stage]])

    def node_stage(self) -> list[int]:
        """node id -> pipeline stage index."""
        out = [0] * self.n
        for stage, c in enumerate(self.order):
            for v in self.members[c]:
                out[v] = stage
        return out

    def to_dict(self) -> dict:
        return {"s": self.s, "sizes": list(self.sizes), "members": [list(m) for m in self.members],
                "order": list(self.order)}

    @classmethod
    def from_dict(cls, d: dict) -> "StageAssignment":
        return cls(s=int(d["s"]), sizes=[int(x) for x in d["sizes"]], members=[[int(v) for v in m] for m in d["members"]],
                   order=[int(x) for x in d["order"]])

    def save(self, path) -> None:
        with open(path, "w") as fh:
            json.dump(self.to_dict(), fh, indent=2, sort_keys=True)
            fh.write("\n")

    @classmethod
    def load(cls, path) -> "StageAssignment":
        with open(path) as fh:
            return cls.from_dict(json.load(fh))

    @classmethod
    def contiguous(cls, sizes: list[int]) -> "StageAssignment":
        """Nodes numbered stage by stage (stage 0 first), identity order: the B200 layout."""
        members, start = [], 0
        for sz in sizes:
            members.append(list(range(start, start + sz)))
            start += sz
        return cls(s=len(sizes), sizes=list(sizes), members=members, order=list(range(len(sizes))))


# ---------------------------------------------------------------------------------------
# GA clustering
# ---------------------------------------------------------------------------------------
@dataclass(frozen=True)
class GAConfig:
    population: int = 64
    generations: int = 500
    mutation_rate: float = 0.3
    tournament: int = 4
    seed: int = 0

    def __post_init__(self):
        if min(self.population, self.generations, self.tournament) < 1:
            raise ValidationError("GA population, generations and tournament size must be positive")
        if not (0 < self.mutation_rate <= 1):
            raise ValidationError(f"GA mutation rate must be in (0, 1], got {self.mutation_rate}")


def _cluster_fitness(perm: np.ndarray, bounds: list[tuple[int, int]], cost: np.ndarray) -> float:
    worst = 0.0
    for a, b in bounds:
        if b - a > 1:
            idx = perm[a:b]
            worst = max(worst, float(cost[np.ix_(idx, idx)].max()))
    return worst


def cluster_nodes(topology: Topology, sizes: list[int], ga_config: GAConfig | None = None,
                  dp_msg_bytes: float = 1.0e8) -> list[list[int]]:
    """Partition nodes into clusters of exactly ``sizes`` minimising the slowest intra-cluster
    pairwise comm_time for a DP-sync message (PAPER.md "bounded by the slowest communication").

    GA: tournament selection, swap-two-nodes-across-clusters mutation, elitism of 1, seeded
    PCG64; deterministic for fixed inputs."""
    cfg = ga_config or GAConfig()
    if any(sz < 1 for sz in sizes) or sum(sizes) != topology.n:
        raise ValidationError(f"cluster sizes {sizes} do not partition n={topology.n} nodes")
    n = topology.n
    cost = comm_matrix(topology, dp_msg_bytes)
    bounds, a = [], 0
    for sz in sizes:
        bounds.append((a, a + sz))
        a += sz
    cluster_of_pos = np.concatenate([np.full(sz, c) for c, sz in enumerate(sizes)])
    rng = np.random.default_rng(cfg.seed)

    pop = [np.arange(n)] + [rng.permutation(n) for _ in range(cfg.population - 1)]
    fit = [_cluster_fitness(p, bounds, cost) for p in pop]
    for _ in range(cfg.generations):
        best = min(range(len(pop)), key=lambda i: (fit[i], i))
        new_pop, new_fit = [pop[best].copy()], [fit[best]]
        while len(new_pop) < cfg.population:
            cand = rng.integers(0, len(pop), size=cfg.tournament)
            win = min(cand.tolist(), key=lambda i: (fit[i], i))
            child = pop[win].copy()
            if len(sizes) > 1 and rng.random() < cfg.mutation_rate:
                i = int(rng.integers(0, n))
                others = np.nonzero(cluster_of_pos != cluster_of_pos[i])[0]
                j = int(others[rng.integers(0, len(others))])
                child[i], child[j] = child[j], child[i]
            new_pop.append(child)
            new_fit.append(_cluster_fitness(child, bounds, cost))
        pop, fit = new_pop, new_fit
    best = min(range(len(pop)), key=lambda i: (fit[i], i))
    members = [sorted(int(v) for v in pop[best][a:b]) for a, b in bounds]
    # canonical form: clusters of equal size are listed by their smallest member id
    by_size: dict[int, list[list[int]]] = {}
    for sz, mem in zip(sizes, members):
        by_size.setdefault(sz, []).append(mem)
    for group in by_size.values():
        group.sort()
    taken = {sz: 0 for sz in by_size}
    out = []
    for sz in sizes:
        out.append(by_size[sz][taken[sz]])
        taken[sz] += 1
    return out


def partition_fitness(topology: Topology, members: list[list[int]], dp_msg_bytes: float = 1.0e8) -> float:
    cost = comm_matrix(topology, dp_msg_bytes)
    worst = 0.0
    for m in members:
        if len(m) > 1:
            worst = max(worst, float(cost[np.ix_(m, m)].max()))
    return worst


# ---------------------------------------------------------------------------------------
# closed-loop TSP over clusters
# ---------------------------------------------------------------------------------------
def stage_distance(topology: Topology, members: list[list[int]], msg_bytes: float) -> np.ndarray:
    """Edge weight between clusters A, B = mean over (a∈A, b∈B) of comm_time(a, b, msg)."""
    cm = comm_matrix(topology, msg_bytes)
    s = len(members)
    w = np.zeros((s, s))
    for a in range(s):
        for b in range(s):
            if a != b:
                w[a, b] = float(cm[np.ix_(members[a], members[b])].mean())
    return w


def solve_closed_tsp(w: np.ndarray, max_s: int = 12) -> tuple[list[int], float]:
    """Exact Held-Karp closed tour from city 0; among optimal tours the lexicographically
    smallest is returned (ties within 1e-9 relative)."""
    s = w.shape[0]
    if s > max_s:
        raise ValidationError(f"exact TSP supports s <= {max_s} stages, got {s}; enable a heuristic solver")
    if s == 1:
        return [0], 0.0
    full = (1 << s) - 1
    # g[mask][j] = cheapest cost to visit the cities not in mask starting at j and return to 0
    g = np.full((1 << s, s), math.inf)
    for j in range(s):
        g[full][j] = w[j, 0]
    for mask in range(full - 1, 0, -1):
        if not mask & 1:
            continue
        for j in range(s):
            if not (mask >> j) & 1:
                continue
            best = math.inf
            for k in range(s):
                if not (mask >> k) & 1:
                    c = w[j, k] + g[mask | (1 << k)][k]
                    if c < best:
                        best = c
            g[mask][j] = best
    opt = g[1][0]
    tour, mask, cur = [0], 1, 0
    while mask != full:
        target = g[mask][cur]
        for k in range(s):
            if (mask >> k) & 1:
                continue
            c = w[cur, k] + g[mask | (1 << k)][k]
            if c <= target + _TIE_EPS * max(1.0, abs(target)):
                tour.append(k)
                mask |= 1 << k
                cur = k
                break
    return tour, float(opt)


def tour_cost(w: np.ndarray, tour: list[int]) -> float:
    return float(sum(w[tour[i], tour[(i + 1) % len(tour)]] for i in range(len(tour))))


def order_stages(topology: Topology, members: list[list[int]], msg_bytes: float) -> StageAssignment:
    """Designate S₀ (the unique largest cluster; cluster 0 on ties), then order the
    clusters by the exact closed-loop TSP, rotated to start at S₀."""
    s = len(members)
    sizes = [len(m) for m in members]
    big = max(sizes)
    s0 = sizes.index(big) if sizes.count(big) == 1 else 0
    # relabel so that S₀ is city 0 of the TSP
    perm = [s0] + [c for c in range(s) if c != s0]
    w = stage_distance(topology, [members[c] for c in perm], msg_bytes)
    tour, _ = solve_closed_tsp(w)
    order = [perm[c] for c in tour]
    return StageAssignment(s=s, sizes=sizes, members=[sorted(m) for m in members], order=order)


def allocate(topology: Topology, s: int, k, msg_bytes: float, ga_config: GAConfig | None = None,
             dp_msg_bytes: float = 1.0e8) -> StageAssignment:
    """stage_sizes -> cluster_nodes -> order_stages."""
    sizes = stage_sizes(topology.n, s, k)
    members = cluster_nodes(topology, sizes, ga_config, dp_msg_bytes)
    return order_stages(topology, members, msg_bytes)
