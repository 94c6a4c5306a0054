"""First-wave microbatch path scheduler: time-dimensioned A* per agent inside a two-phase
conflict-based search (§3.3-3.4 and Algorithm 2).

Phase 1 (``find_candidates``) collects up to ``pool_size`` CBS nodes whose paths satisfy CC1,
CC2 and CC3 (H1 "32 in our experiments", H2 slow-agent exemption).  Phase 2
(``resolve_throughput``) resolves TC1 (≤ m paths per node) then TC2 (no overlapping planned
compute on a node), critical path first, with the H3 single-child rule; if the pool is
exhausted the conflict-minimal node seen is returned flagged unresolved.

Ambiguities of the spec are pinned here and in DESIGN.md:
* agent a starts at S₀ node ``s0_nodes[a % |S₀|]`` (m agents per S₀ node);
* CC2: the visited stage sequence has at most one descent, and transposing that adjacent pair
  gives a strictly increasing sequence;
* CC3 cap = ⌈|𝒫|·(l−1)/(s−1)⌉ visits per non-first stage;
* a CC3 conflict branches into up to ``cc3_branching`` children: the paper's choice (the K−cap
  fastest non-exempt offending paths) first, then the next subsets in lexicographic order of
  speed rank — without branching phase 1 is a single chain and can never fill a pool;
* planned compute intervals used for TC2 are the forward ones (backward collisions are left to
  the simulator); an agent's own interval constraints also delay its backward;
* heap ties: A* (cost, agent, node, time, node-sequence); CBS (cost, Σe2e, |constraints|, id).
"""

from __future__ import annotations

import ctypes
import heapq
import itertools
import json
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from fractions import Fraction

import numpy as np

from .allocation import StageAssignment
from .errors import InfeasibleError, ValidationError
from .topology import Topology, comm_matrix

INF = math.inf


# ---------------------------------------------------------------------------------------
# domain types
# ---------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Agent:
    id: int
    origin: int


@dataclass(frozen=True, order=True)
class IntervalConstraint:
    """Agent ``agent`` may not compute on ``node`` during [t_start, t_end] (Algorithm 2)."""

    agent: int
    node: int
    t_start: float
    t_end: float

    def __post_init__(self):
        if not self.t_start < self.t_end:
            raise ValidationError(f"constraint interval must satisfy t_start < t_end, got [{self.t_start}, {self.t_end}]")

    @property
    def permanent(self) -> bool:
        return self.t_start == -INF and self.t_end == INF

    def to_dict(self) -> dict:
        return {"agent": self.agent, "node": self.node, "t_start": _jf(self.t_start), "t_end": _jf(self.t_end)}

    @classmethod
    def from_dict(cls, d: dict) -> "IntervalConstraint":
        return cls(int(d["agent"]), int(d["node"]), _pf(d["t_start"]), _pf(d["t_end"]))


def _jf(x: float):
    return "-inf" if x == -INF else ("inf" if x == INF else x)


def _pf(x) -> float:
    return float(x)


@dataclass(frozen=True)
class Visit:
    node: int
    stage: int
    arrival: float
    start: float
    end: float


@dataclass(frozen=True)
class PathPlan:
    """One agent's timed forward route origin → … → origin, plus the mirrored backward plan."""

    agent: int
    visits: tuple[Visit, ...]        # forward computes, then the return visit at the origin
    bwd_visits: tuple[Visit, ...]    # backward computes in execution order (last stage first)
    swap_count: int
    e2e: float

    @property
    def origin(self) -> int:
        return self.visits[0].node

    @property
    def nodes(self) -> tuple[int, ...]:
        """Forward compute nodes in path order (origin first, return visit excluded)."""
        return tuple(v.node for v in self.visits[:-1])

    @property
    def stages(self) -> tuple[int, ...]:
        return tuple(v.stage for v in self.visits[:-1])

    def fwd_intervals(self):
        return [(v.node, v.start, v.end) for v in self.visits[:-1]]

    def to_dict(self) -> dict:
        enc = lambda v: [v.node, v.stage, v.arrival, v.start, v.end]  # noqa: E731
        return {"agent": self.agent, "visits": [enc(v) for v in self.visits],
                "bwd_visits": [enc(v) for v in self.bwd_visits], "swap_count": self.swap_count, "e2e": self.e2e}

    @classmethod
    def from_dict(cls, d: dict) -> "PathPlan":
        dec = lambda r: Visit(int(r[0]), int(r[1]), float(r[2]), float(r[3]), float(r[4]))  # noqa: E731
        return cls(int(d["agent"]), tuple(dec(r) for r in d["visits"]), tuple(dec(r) for r in d["bwd_visits"]),
                   int(d["swap_count"]), float(d["e2e"]))


@dataclass(frozen=True)
class SchedulerConfig:
    k: float = 25.0
    msg_bytes: float = 8_388_608.0
    pool_size: int = 32
    slow_exempt_fraction: float = 0.25
    delta_tie: float = 1.0
    max_swaps: int = 1
    cc3_branching: int = 4
    resolve_tc2: bool = True
    max_expansions: int = 4000
    # B200 extension (not in SPEC): agents whose path must contain exactly one swap.  On a uniform
    # NVSwitch box a swap never lowers a path's cost, so A* (ties to the lowest stage) never picks
    # one; listing agents here makes a config exercise reordered paths (BASELINE configs[2]).
    swap_agents: tuple = ()
    # Extension (not in SPEC): the throughput phase removes *planned* first-wave collisions, which
    # can cost more (longer paths) than the collisions would have; when it ends unresolved its
    # conflict-minimal node is not the fastest one either.  With sim_select = W > 0
    # schedule() keeps, by simulated iteration (W waves of the agents), the faster of the phase's
    # answer and the TC1-only resolution of the same pool (SkipPipe-without-TC2's answer) -- when
    # unresolved, also the TC1-clean nodes the search met -- then descends greedily over the
    # remaining collisions.  0 = Algorithm 1 only (the B200 run configs use 0: on one NVSwitch box
    # TC2 changes nothing measurable, and their plans are the GPU-validated ones).
    sim_select: int = int(os.environ.get("SPX_SCHED_SIM_SELECT", "4"))
    sim_microbatches: int = 0  # microbatches of the selection's simulation (0: sim_select waves)

    def __post_init__(self):
        if self.pool_size < 1:
            raise ValidationError("pool_size must be >= 1")
        if not (0 <= self.slow_exempt_fraction < 1):
            raise ValidationError("slow_exempt_fraction must be in [0, 1)")
        if self.delta_tie < 0:
            raise ValidationError("delta_tie must be >= 0")
        if self.max_swaps != 1:
            raise ValidationError("max_swaps is fixed at 1 (multiple swaps are a non-goal, SPEC.md:314)")
        if not self.msg_bytes > 0:
            raise ValidationError("msg_bytes must be positive")
        if self.sim_select < 0 or self.sim_microbatches < 0:
            raise ValidationError("sim_select and sim_microbatches must be >= 0")
        object.__setattr__(self, "swap_agents", tuple(sorted(int(a) for a in self.swap_agents)))

    def to_dict(self) -> dict:
        return {"k": self.k, "msg_bytes": self.msg_bytes, "pool_size": self.pool_size,
                "slow_exempt_fraction": self.slow_exempt_fraction, "delta_tie": self.delta_tie,
                "max_swaps": self.max_swaps, "cc3_branching": self.cc3_branching, "resolve_tc2": self.resolve_tc2,
                "max_expansions": self.max_expansions, "swap_agents": list(self.swap_agents),
                "sim_select": self.sim_select, "sim_microbatches": self.sim_microbatches}

    @classmethod
    def from_dict(cls, d: dict) -> "SchedulerConfig":
        return cls(**d)


@dataclass
class SearchNode:
    constraints: frozenset
    paths: dict  # agent id -> PathPlan
    cost: float
    uid: int = 0

    @property
    def sum_e2e(self) -> float:
        return float(sum(p.e2e for p in self.paths.values()))

    def key(self):
        return (self.cost, self.sum_e2e, len(self.constraints), self.uid)

    def signature(self):
        return tuple((a, self.paths[a].nodes) for a in sorted(self.paths))


# conflicts --------------------------------------------------------------------------------
@dataclass(frozen=True)
class StageOveruse:
    stage: int
    count: int
    cap: int


@dataclass(frozen=True)
class NodeOveruse:
    node: int
    count: int
    m: int


@dataclass(frozen=True)
class Collision:
    path_i: int
    path_j: int
    node: int
    overlap: tuple[float, float]
    interval_i: tuple[float, float]
    interval_j: tuple[float, float]


# ---------------------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------------------
def path_length(s: int, k) -> int:
    """l = s·(100 − k)/100 visited stages incl. S₀; must be integral."""
    kf = k if isinstance(k, Fraction) else Fraction(k).limit_denominator(10**6)
    l_ = Fraction(s) * (100 - kf) / 100
    if l_.denominator != 1 or l_ < 1:
        raise ValidationError(f"s={s}, k={float(kf):g} gives a non-integral path length {float(l_):g}")
    return int(l_)


def cc3_cap(n_agents: int, s: int, l: int) -> int:
    return math.ceil(n_agents * (l - 1) / (s - 1)) if s > 1 else 0


def make_agents(assignment: StageAssignment, m: int) -> list[Agent]:
    """|𝒫| = m·|S₀| agents; agent a starts at S₀ node a mod |S₀|."""
    s0 = assignment.stage_nodes(0)
    return [Agent(a, s0[a % len(s0)]) for a in range(m * len(s0))]


def cc2_extend(seq: tuple[int, ...], swaps: int, x: int, max_swaps: int = 1):
    """Return the swap count after appending stage x to seq, or None if CC2 forbids it."""
    if x in seq:
        return None
    if x > max(seq):
        return swaps
    if swaps >= max_swaps or len(seq) < 2:
        return None
    if seq[-2] < x < seq[-1]:
        return swaps + 1
    return None


class _Timing:
    """Per-node compute and pairwise comm times for one scheduling problem."""

    def __init__(self, topology: Topology, msg_bytes: float):
        self.fwd = topology.compute_fwd_ms.astype(float)
        self.bwd = self.fwd * float(topology.bwd_ratio)
        self.comm = comm_matrix(topology, msg_bytes)
        self._native = {}

    def native_problem(self, assignment: StageAssignment, l: int, max_swaps: int):
        """The spx_sched_problem struct for libspx_sched (arrays kept alive on this object)."""
        key = (tuple(assignment.node_stage()), l, max_swaps)
        if key not in self._native:
            ns = np.ascontiguousarray(assignment.node_stage(), dtype=np.int32)
            fwd = np.ascontiguousarray(self.fwd, dtype=np.float64)
            bwd = np.ascontiguousarray(self.bwd, dtype=np.float64)
            comm = np.ascontiguousarray(self.comm, dtype=np.float64)
            st = _SchedProblem(len(ns), assignment.s, l, max_swaps, ns.ctypes.data_as(_PI32),
                               fwd.ctypes.data_as(_PF64), bwd.ctypes.data_as(_PF64), comm.ctypes.data_as(_PF64))
            self._native[key] = (st, ns, fwd, bwd, comm)
        return self._native[key][0]


# ---------------------------------------------------------------------------------------
# native planner (libspx_sched.so, include/spx_sched.h)
# ---------------------------------------------------------------------------------------
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PF64 = ctypes.POINTER(ctypes.c_double)


class _SchedProblem(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("s", ctypes.c_int32), ("l", ctypes.c_int32), ("max_swaps", ctypes.c_int32),
                ("node_stage", _PI32), ("fwd", _PF64), ("bwd", _PF64), ("comm", _PF64)]


_SCHED_LIB: list = []


def native_lib():
    """libspx_sched.so, or None when it is not built or SPX_SCHED_NATIVE=0 (Python planner).
    Both planners give identical schedules (tests/test_scheduler_native.py)."""
    if os.environ.get("SPX_SCHED_NATIVE", "1") == "0":
        return None
    if not _SCHED_LIB:
        path = Path(__file__).resolve().parent / "libspx_sched.so"
        lib = None
        if path.exists():
            lib = ctypes.CDLL(str(path))
            lib.spx_sched_astar.argtypes = [ctypes.POINTER(_SchedProblem), ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, _PI32, _PF64, _PF64, _PI32, _PF64, _PF64, _PI32, _PI32,
                                            _PF64]
            lib.spx_sched_collisions.restype = ctypes.c_int64
            lib.spx_sched_collisions.argtypes = [ctypes.c_int32, _PI32, _PI32, _PI32, _PF64, _PF64, ctypes.c_int32,
                                                 ctypes.c_int64, _PI32, _PF64]
        _SCHED_LIB.append(lib)
    return _SCHED_LIB[0]


def _astar_native(lib, agent: Agent, assignment: StageAssignment, l: int, constraints, config, tm: _Timing):
    node_stage = assignment.node_stage()
    mine = [c for c in constraints if c.agent == agent.id]
    if any(c.permanent and c.node == agent.origin for c in mine):
        raise InfeasibleError(f"agent {agent.id}: origin {agent.origin} is banned")
    k = len(mine)
    cn = (ctypes.c_int32 * max(1, k))(*[c.node for c in mine])
    c0 = (ctypes.c_double * max(1, k))(*[c.t_start for c in mine])
    c1 = (ctypes.c_double * max(1, k))(*[c.t_end for c in mine])
    s = assignment.s
    nodes = (ctypes.c_int32 * s)()
    fw = (ctypes.c_double * (3 * (s + 1)))()
    bw = (ctypes.c_double * (3 * s))()
    ln, sw, e2e = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
    rc = lib.spx_sched_astar(ctypes.byref(tm.native_problem(assignment, l, config.max_swaps)), agent.origin,
                             int(agent.id in config.swap_agents), k, cn, c0, c1, nodes, fw, bw, ctypes.byref(ln),
                             ctypes.byref(sw), ctypes.byref(e2e))
    if rc == 1:
        raise InfeasibleError(f"agent {agent.id}: no path satisfies its {k} constraints")
    if rc != 0:
        raise ValidationError(f"spx_sched_astar: bad arguments (rc={rc})")
    n_ = ln.value
    route = [nodes[i] for i in range(n_)]
    visits = tuple(Visit(v, node_stage[v], fw[3 * i], fw[3 * i + 1], fw[3 * i + 2]) for i, v in enumerate(route))
    visits += (Visit(agent.origin, 0, fw[3 * n_], fw[3 * n_ + 1], fw[3 * n_ + 2]),)
    back = list(reversed(route[1:])) + [agent.origin]
    bwd = tuple(Visit(v, node_stage[v] if i < n_ - 1 else 0, bw[3 * i], bw[3 * i + 1], bw[3 * i + 2])
                for i, v in enumerate(back))
    return PathPlan(agent.id, visits, bwd, sw.value, e2e.value)


def _earliest_start(windows: list[tuple[float, float]], t: float, dur: float) -> float:
    """Smallest t' ≥ t such that [t', t'+dur) overlaps no window (deferred to the window's end)."""
    moved = True
    while moved:
        moved = False
        for ts, te in windows:
            if t < te and ts < t + dur:
                t = te
                moved = True
    return t


# ---------------------------------------------------------------------------------------
# A* (uniform cost, h = 0, no closed set)
# ---------------------------------------------------------------------------------------
def astar_path(agent: Agent, topology: Topology, assignment: StageAssignment, constraints, config: SchedulerConfig,
               timing: _Timing | None = None) -> PathPlan:
    """Minimum-e2e PathPlan for one agent under CC1, CC2, exact-l and its interval constraints.

    States are (node, visited stages, swap count, time).  Entering a constrained interval is
    deferred to the interval's end.  Once l stages are visited the origin is re-enqueued with a
    completion flag keyed by the forward+backward e2e; popping a flagged state returns it
    (PAPER.md:245-267)."""
    tm = timing or _Timing(topology, config.msg_bytes)
    s = assignment.s
    l = path_length(s, config.k)
    node_stage = assignment.node_stage()
    stage_nodes = [assignment.stage_nodes(i) for i in range(s)]
    if node_stage[agent.origin] != 0:
        raise ValidationError(f"agent {agent.id} origin {agent.origin} is not in S0", row=agent.id)

    lib = native_lib()
    if lib is not None:
        return _astar_native(lib, agent, assignment, l, constraints, config, tm)

    banned: set[int] = set()
    windows: dict[int, list[tuple[float, float]]] = {}
    for c in constraints:
        if c.agent != agent.id:
            continue
        if c.permanent:
            banned.add(c.node)
        else:
            windows.setdefault(c.node, []).append((c.t_start, c.t_end))
    for w in windows.values():
        w.sort()
    if agent.origin in banned:
        raise InfeasibleError(f"agent {agent.id}: origin {agent.origin} is banned")

    def start_at(node, t, dur):
        w = windows.get(node)
        return _earliest_start(w, t, dur) if w else t

    def backward(nodes: tuple[int, ...], t_ret: float):
        out = []
        t = t_ret
        prev = agent.origin
        for v in reversed(nodes[1:]):
            arr = t + tm.comm[prev, v]
            st = start_at(v, arr, tm.bwd[v])
            t = st + tm.bwd[v]
            out.append(Visit(v, node_stage[v], arr, st, t))
            prev = v
        arr = t + (tm.comm[prev, agent.origin] if prev != agent.origin else 0.0)
        st = start_at(agent.origin, arr, tm.bwd[agent.origin])
        t = st + tm.bwd[agent.origin]
        out.append(Visit(agent.origin, 0, arr, st, t))
        return tuple(out), t

    o = agent.origin
    st0 = start_at(o, 0.0, tm.fwd[o])
    first = Visit(o, 0, 0.0, st0, st0 + tm.fwd[o])
    heap: list = []
    # entry: (cost, agent, node, time, nodes, flagged, payload)
    heapq.heappush(heap, (first.end, agent.id, o, first.end, (o,), 0, ((0,), 0, (first,))))
    while heap:
        cost, _, u, t, nodes, flagged, payload = heapq.heappop(heap)
        if flagged:
            fwd_visits, bwd_visits, swaps = payload
            return PathPlan(agent.id, fwd_visits, bwd_visits, swaps, cost)
        seq, swaps, visits = payload
        if len(seq) == l:
            if swaps == 0 and agent.id in config.swap_agents:
                continue
            t_ret = t + (tm.comm[u, o] if u != o else 0.0)
            ret = Visit(o, 0, t_ret, t_ret, t_ret)
            bwd_visits, e2e = backward(nodes, t_ret)
            heapq.heappush(heap, (e2e, agent.id, o, t_ret, nodes, 1, (visits + (ret,), bwd_visits, swaps)))
            continue
        for x in range(1, s):
            ns = cc2_extend(seq, swaps, x, config.max_swaps)
            if ns is None:
                continue
            for v in stage_nodes[x]:
                if v in banned:
                    continue
                arr = t + tm.comm[u, v]
                st = start_at(v, arr, tm.fwd[v])
                end = st + tm.fwd[v]
                vis = Visit(v, x, arr, st, end)
                heapq.heappush(heap, (end, agent.id, v, end, nodes + (v,), 0, (seq + (x,), ns, visits + (vis,))))
    raise InfeasibleError(f"agent {agent.id}: no path satisfies its {sum(1 for c in constraints if c.agent == agent.id)} constraints")


def time_fixed_path(agent_id: int, nodes: list[int], topology: Topology, assignment: StageAssignment,
                    msg_bytes: float) -> PathPlan:
    """Contention-free PathPlan of a given node sequence (used by the baselines)."""
    tm = _Timing(topology, msg_bytes)
    node_stage = assignment.node_stage()
    o = nodes[0]
    visits, t, prev = [], 0.0, None
    for v in nodes:
        arr = 0.0 if prev is None else t + tm.comm[prev, v]
        visits.append(Visit(v, node_stage[v], arr, arr, arr + tm.fwd[v]))
        t = arr + tm.fwd[v]
        prev = v
    t_ret = t + (tm.comm[prev, o] if prev != o else 0.0)
    visits.append(Visit(o, 0, t_ret, t_ret, t_ret))
    bwd, t, prev = [], t_ret, o
    for v in reversed(nodes[1:]):
        arr = t + tm.comm[prev, v]
        bwd.append(Visit(v, node_stage[v], arr, arr, arr + tm.bwd[v]))
        t, prev = arr + tm.bwd[v], v
    arr = t + (tm.comm[prev, o] if prev != o else 0.0)
    bwd.append(Visit(o, 0, arr, arr, arr + tm.bwd[o]))
    stages = [node_stage[v] for v in nodes]
    swaps = sum(1 for i in range(1, len(stages)) if stages[i] < stages[i - 1])
    return PathPlan(agent_id, tuple(visits), tuple(bwd), swaps, arr + tm.bwd[o])


# ---------------------------------------------------------------------------------------
# conflicts
# ---------------------------------------------------------------------------------------
def stage_visit_counts(paths: dict, assignment: StageAssignment) -> list[int]:
    counts = [0] * assignment.s
    for p in paths.values():
        for st in set(p.stages):
            counts[st] += 1
    return counts


def node_path_counts(paths: dict, n: int) -> list[int]:
    counts = [0] * n
    for p in paths.values():
        for v in set(p.nodes):
            counts[v] += 1
    return counts


def critical_agent(paths: dict) -> int:
    return min(paths, key=lambda a: (-paths[a].e2e, a))


def detect_conflicts(node: SearchNode, topology: Topology, assignment: StageAssignment, m: int, cap: int | None = None,
                     k=None) -> list:
    """Typed conflicts ordered StageOveruse (by stage), NodeOveruse (by node), Collision
    (critical-path first, then overlap start) — SPEC.md:268-276."""
    paths = node.paths
    out: list = []
    if cap is None and k is not None:
        cap = cc3_cap(len(paths), assignment.s, path_length(assignment.s, k))
    if cap is not None:
        for st, c in enumerate(stage_visit_counts(paths, assignment)):
            if st >= 1 and c > cap:
                out.append(StageOveruse(st, c, cap))
    for v, c in enumerate(node_path_counts(paths, topology.n)):
        if c > m:
            out.append(NodeOveruse(v, c, m))
    crit = critical_agent(paths) if paths else -1
    lib = native_lib()
    if lib is not None and paths:
        cols = _collisions_native(lib, paths, topology.n)
        cols.sort(key=lambda c: (0 if crit in (c.path_i, c.path_j) else 1, c.overlap[0], c.node, c.path_i, c.path_j))
        return out + cols
    by_node: dict[int, list] = {}
    for a in sorted(paths):
        for v, s0, e0 in paths[a].fwd_intervals():
            by_node.setdefault(v, []).append((a, s0, e0))
    cols = []
    for v in sorted(by_node):
        iv = by_node[v]
        for (a, s1, e1), (b, s2, e2) in itertools.combinations(iv, 2):
            if a == b:
                continue
            lo, hi = max(s1, s2), min(e1, e2)
            if lo < hi:
                i, j = (a, b) if a < b else (b, a)
                ii, jj = ((s1, e1), (s2, e2)) if a < b else ((s2, e2), (s1, e1))
                cols.append(Collision(i, j, v, (lo, hi), ii, jj))
    cols.sort(key=lambda c: (0 if crit in (c.path_i, c.path_j) else 1, c.overlap[0], c.node, c.path_i, c.path_j))
    return out + cols


def _collisions_native(lib, paths: dict, n: int) -> list:
    agents = sorted(paths)
    ivs = [paths[a].fwd_intervals() for a in agents]
    tot = sum(len(x) for x in ivs)
    ids = (ctypes.c_int32 * len(agents))(*agents)
    cnt = (ctypes.c_int32 * len(agents))(*[len(x) for x in ivs])
    vn = (ctypes.c_int32 * tot)(*[v for x in ivs for v, _, _ in x])
    vs = (ctypes.c_double * tot)(*[s0 for x in ivs for _, s0, _ in x])
    ve = (ctypes.c_double * tot)(*[e0 for x in ivs for _, _, e0 in x])
    cap = 64
    while True:
        ijn = (ctypes.c_int32 * (3 * cap))()
        tms = (ctypes.c_double * (6 * cap))()
        found = lib.spx_sched_collisions(len(agents), ids, cnt, vn, vs, ve, n, cap, ijn, tms)
        if found < 0:
            raise ValidationError("spx_sched_collisions: bad arguments")
        if found <= cap:
            break
        cap = int(found)
    return [Collision(ijn[3 * i], ijn[3 * i + 1], ijn[3 * i + 2], (tms[6 * i], tms[6 * i + 1]),
                      (tms[6 * i + 2], tms[6 * i + 3]), (tms[6 * i + 4], tms[6 * i + 5])) for i in range(found)]


# ---------------------------------------------------------------------------------------
# CBS
# ---------------------------------------------------------------------------------------
class _Planner:
    def __init__(self, topology, assignment, config):
        self.topology, self.assignment, self.config = topology, assignment, config
        self.timing = _Timing(topology, config.msg_bytes)
        self.agents = {a.id: a for a in make_agents(assignment, topology.mem_capacity)}
        self.uid = itertools.count()
        self._plans: dict = {}  # (agent, its constraints) -> PathPlan or InfeasibleError

    def plan(self, aid: int, constraints) -> PathPlan:
        """astar_path for one agent, memoised on the constraints that concern it (CBS children
        re-plan the same agent under the same constraint set many times); deterministic."""
        key = (aid, frozenset(c for c in constraints if c.agent == aid))
        hit = self._plans.get(key)
        if hit is None:
            try:
                hit = astar_path(self.agents[aid], self.topology, self.assignment, key[1], self.config, self.timing)
            except InfeasibleError as e:
                hit = e
            self._plans[key] = hit
        if isinstance(hit, InfeasibleError):
            raise hit
        return hit

    def root(self) -> SearchNode:
        paths = {a: self.plan(a, ()) for a in sorted(self.agents)}
        return self.make(frozenset(), paths)

    def make(self, constraints, paths) -> SearchNode:
        return SearchNode(constraints, paths, max(p.e2e for p in paths.values()), next(self.uid))

    def child(self, parent: SearchNode, new: list[IntervalConstraint]):
        cons = parent.constraints | frozenset(new)
        if cons == parent.constraints:
            return None
        paths = dict(parent.paths)
        try:
            for aid in sorted({c.agent for c in new}):
                paths[aid] = self.plan(aid, cons)
        except InfeasibleError:
            return None
        return self.make(cons, paths)


def _exempt(paths: dict, fraction: float) -> set[int]:
    n_ex = math.ceil(len(paths) * fraction)
    slow = sorted(paths, key=lambda a: (-round(paths[a].e2e, 9), a))
    return set(slow[:n_ex])


def _fastest(paths: dict, agents, constraints=()) -> list[int]:
    """Agents by e2e ascending.  Ties (common on uniform topologies, where every path of the same
    length costs the same) go to the agent with fewer permanent bans, then the lower id — so the
    skip budget is spread over agents instead of exhausting one agent's."""
    bans: dict[int, int] = {}
    for c in constraints:
        if c.permanent:
            bans[c.agent] = bans.get(c.agent, 0) + 1
    return sorted(agents, key=lambda a: (round(paths[a].e2e, 9), bans.get(a, 0), a))


def _cc3_children(pl, node: SearchNode, st: int, cap: int, config: SchedulerConfig,
                  assignment: StageAssignment) -> list[SearchNode]:
    """Branch on a CC3 conflict at stage ``st``: ban every node of the stage for K−cap of the
    offending paths — the fastest non-exempt ones first (Algorithm 2, H2), then further subsets."""
    offending = [a for a in node.paths if st in node.paths[a].stages]
    exempt = _exempt(node.paths, config.slow_exempt_fraction)
    cand = _fastest(node.paths, [a for a in offending if a not in exempt], node.constraints)
    need = min(len(offending) - cap, len(cand))
    out = []
    if need <= 0:
        return out
    for combo in itertools.islice(itertools.combinations(cand, need), max(1, config.cc3_branching)):
        ch = pl.child(node, [IntervalConstraint(a, v, -INF, INF) for a in combo for v in assignment.stage_nodes(st)])
        if ch is not None:
            out.append(ch)
    return out


def find_candidates(topology: Topology, assignment: StageAssignment, agents, config: SchedulerConfig,
                    _planner: _Planner | None = None) -> list[SearchNode]:
    """Phase 1: best-first CBS until ``pool_size`` CC3-feasible nodes are collected (H1, H2)."""
    pl = _planner or _Planner(topology, assignment, config)
    if agents is not None:
        pl.agents = {a.id: a for a in agents}
    l = path_length(assignment.s, config.k)
    cap = cc3_cap(len(pl.agents), assignment.s, l)
    root = pl.root()
    open_: list = [(root.key(), root)]
    pool, seen_sig, seen_cons = [], set(), {root.constraints}
    expansions = 0
    while open_ and len(pool) < config.pool_size and expansions < config.max_expansions:
        _, node = heapq.heappop(open_)
        expansions += 1
        counts = stage_visit_counts(node.paths, assignment)
        over = [st for st in range(1, assignment.s) if counts[st] > cap]
        if not over:
            sig = node.signature()
            if sig not in seen_sig:
                seen_sig.add(sig)
                pool.append(node)
            continue
        children = []
        for ch in _cc3_children(pl, node, over[0], cap, config, assignment):
            if ch.constraints not in seen_cons:
                seen_cons.add(ch.constraints)
                children.append(ch)
        for ch in children:
            heapq.heappush(open_, (ch.key(), ch))
    if not pool:
        raise InfeasibleError("phase 1 exhausted without a CC3-feasible candidate")
    return pool


SIM_SELECT_MAX = 256    # TC1-clean nodes scored by simulation per resolve_throughput call
SIM_REFINE_STEPS = 32   # greedy collision-resolution steps after the search (sim_select)
SIM_REFINE_FANOUT = 16  # collisions tried per step, critical path first


class _SimScorer:
    """Simulated iteration makespan of a search node (SchedulerConfig.sim_select waves of the
    node's agents), memoised per constraint set (a node's paths are a function of it)."""

    def __init__(self, topology: Topology, config: SchedulerConfig, pl: "_Planner"):
        from .simulator import SimConfig, simulate
        self._simulate = simulate
        self.topology, self.config = topology, config
        self.agents = [pl.agents[a] for a in sorted(pl.agents)]
        M = config.sim_microbatches or len(self.agents) * config.sim_select
        self.sc = SimConfig(total_microbatches=M, msg_bytes=config.msg_bytes)
        self.memo: dict = {}

    def __call__(self, nd: SearchNode) -> float:
        t = self.memo.get(nd.constraints)
        if t is None:
            sch = Schedule(self.config, self.agents, dict(nd.paths), sorted(nd.constraints), nd.cost, False)
            t = self.memo[nd.constraints] = self._simulate(sch, self.topology, self.sc).iteration_makespan
        return t


def _sim_refine(node: SearchNode, score: _SimScorer, pl: "_Planner", topology: Topology,
                assignment: StageAssignment, cap: int) -> SearchNode:
    """Greedy simulated descent over TC2 resolutions: try both children of each of the first
    SIM_REFINE_FANOUT collisions (the faster path avoids the slower one's window, or the reverse),
    keep the child with the shortest simulated iteration if it beats the current node without
    adding TC1 / CC3 conflicts; repeat."""
    m = topology.mem_capacity
    cur, t_cur = node, score(node)
    def other(cs):  # (CC3, TC1) conflict counts
        return (sum(isinstance(x, StageOveruse) for x in cs), sum(isinstance(x, NodeOveruse) for x in cs))

    for _ in range(SIM_REFINE_STEPS):
        conf = detect_conflicts(cur, topology, assignment, m, cap=cap)
        colls = [c for c in conf if isinstance(c, Collision)]
        if not colls:
            break
        n_other = other(conf)
        best, t_best = None, t_cur
        for c in colls[:SIM_REFINE_FANOUT]:
            for agent, iv in ((c.path_j, c.interval_i), (c.path_i, c.interval_j)):
                ch = pl.child(cur, [IntervalConstraint(agent, c.node, *iv)])
                if ch is None:
                    continue
                o = other(detect_conflicts(ch, topology, assignment, m, cap=cap))
                if o[0] > n_other[0] or o[1] > n_other[1]:
                    continue
                t = score(ch)
                if t < t_best:
                    best, t_best = ch, t
        if best is None:
            break
        cur, t_cur = best, t_best
    return cur


def resolve_throughput(candidates: list[SearchNode], topology: Topology, assignment: StageAssignment,
                       config: SchedulerConfig, _planner: _Planner | None = None) -> tuple[SearchNode, bool]:
    """Phase 2: resolve TC1 then TC2 (critical path first, H3).  Returns (node, resolved)."""
    if not candidates:
        raise ValidationError("resolve_throughput needs a non-empty candidate list")
    pl = _planner or _Planner(topology, assignment, config)
    m = topology.mem_capacity
    cap = cc3_cap(len(candidates[0].paths), assignment.s, path_length(assignment.s, config.k))
    open_ = [(c.key(), c) for c in candidates]
    heapq.heapify(open_)
    seen_cons = {c.constraints for c in candidates}
    best, best_key = None, None
    expansions = 0
    # SchedulerConfig.sim_select: TC1-clean nodes met on the way are scored by simulated iteration
    # (at most SIM_SELECT_MAX of them); when the search ends unresolved, the best one replaces the
    # conflict-minimal answer if it is faster
    sim_on = bool(config.sim_select) and config.resolve_tc2
    scored: list = []  # (makespan, order, node)
    sim_time = _SimScorer(topology, config, pl) if sim_on else None

    def finish(node, resolved):
        if resolved or not scored:  # a fully resolved node is Algorithm 1's answer, kept as is
            return node, resolved
        t_node = sim_time(node)
        t_best, _, nd = min(scored, key=lambda x: (x[0], x[1]))
        if t_best < t_node:
            return nd, not detect_conflicts(nd, topology, assignment, m, cap=cap)
        return node, resolved

    while open_ and expansions < config.max_expansions:
        _, node = heapq.heappop(open_)
        expansions += 1
        conf = [c for c in detect_conflicts(node, topology, assignment, m, cap=cap)
                if not isinstance(c, Collision) or config.resolve_tc2]
        k = (any(isinstance(c, StageOveruse) for c in conf), len(conf), node.key())
        if best is None or k < best_key:
            best, best_key = node, k
        if sim_on and conf and len(scored) < SIM_SELECT_MAX and all(isinstance(c, Collision) for c in conf):
            scored.append((sim_time(node), len(scored), node))
        if not conf:
            return finish(node, True)
        c = conf[0]
        children = []
        if isinstance(c, StageOveruse):
            # a TC1/TC2 re-route broke CC3: restore it first (SPEC.md:290 holds for every output)
            children.extend(_cc3_children(pl, node, c.stage, cap, config, assignment))
        elif isinstance(c, NodeOveruse):
            # the slowest path through the node is exempt; the paper's child bans the K−m fastest,
            # further children (cc3_branching) ban the next subsets in speed-rank order
            through = _fastest(node.paths, [a for a in node.paths if c.node in node.paths[a].nodes], node.constraints)
            for combo in itertools.islice(itertools.combinations(through[:-1], c.count - c.m),
                                          max(1, config.cc3_branching)):
                children.append(pl.child(node, [IntervalConstraint(a, c.node, -INF, INF) for a in combo]))
        else:
            ei, ej = node.paths[c.path_i].e2e, node.paths[c.path_j].e2e
            tie = abs(ei - ej) < config.delta_tie
            if ei > ej or tie:   # p_j (faster) avoids p_i's window
                children.append(pl.child(node, [IntervalConstraint(c.path_j, c.node, *c.interval_i)]))
            if ei < ej or tie:
                children.append(pl.child(node, [IntervalConstraint(c.path_i, c.node, *c.interval_j)]))
        for ch in children:
            if ch is not None and ch.constraints not in seen_cons:
                seen_cons.add(ch.constraints)
                heapq.heappush(open_, (ch.key(), ch))
    return finish(best, False)


# ---------------------------------------------------------------------------------------
# end to end
# ---------------------------------------------------------------------------------------
@dataclass
class Schedule:
    config: SchedulerConfig
    agents: list[Agent]
    paths: dict          # agent id -> PathPlan
    constraints: list
    cost_ms: float
    resolved: bool
    kind: str = "SkipPipe"

    def path_nodes(self) -> dict[int, tuple[int, ...]]:
        return {a: p.nodes for a, p in self.paths.items()}

    def to_dict(self) -> dict:
        return {
            "kind": self.kind,
            "config": self.config.to_dict(),
            "agents": [{"id": a.id, "origin": a.origin} for a in self.agents],
            "paths": [self.paths[a.id].to_dict() for a in self.agents],
            "constraints": [c.to_dict() for c in sorted(self.constraints)],
            "cost_ms": self.cost_ms,
            "resolved": self.resolved,
        }

    @classmethod
    def from_dict(cls, d: dict) -> "Schedule":
        agents = [Agent(int(a["id"]), int(a["origin"])) for a in d["agents"]]
        paths = {}
        for p in d["paths"]:
            pp = PathPlan.from_dict(p)
            paths[pp.agent] = pp
        return cls(SchedulerConfig.from_dict(d["config"]), agents, paths,
                   [IntervalConstraint.from_dict(c) for c in d["constraints"]], float(d["cost_ms"]), bool(d["resolved"]),
                   d.get("kind", "SkipPipe"))

    def dumps(self) -> str:
        return json.dumps(self.to_dict(), indent=2, sort_keys=True) + "\n"

    def save(self, path) -> None:
        with open(path, "w") as fh:
            fh.write(self.dumps())

    @classmethod
    def load(cls, path) -> "Schedule":
        with open(path) as fh:
            return cls.from_dict(json.load(fh))


def schedule(topology: Topology, assignment: StageAssignment, config: SchedulerConfig) -> Schedule:
    """Algorithm 1: find_candidates then resolve_throughput; deterministic for fixed inputs."""
    if assignment.n != topology.n:
        raise ValidationError(f"assignment covers {assignment.n} nodes, topology has {topology.n}")
    pl = _Planner(topology, assignment, config)
    agents = [pl.agents[a] for a in sorted(pl.agents)]
    pool = find_candidates(topology, assignment, None, config, pl)
    node, resolved = resolve_throughput(pool, topology, assignment, config, pl)
    if config.sim_select and config.resolve_tc2:
        # candidate selection by simulated iteration (SchedulerConfig.sim_select): the TC1-only
        # resolution of the same pool (what SkipPipe-without-TC2 returns) against the TC2 result,
        # then a greedy simulated descent over the remaining collisions
        score = _SimScorer(topology, config, pl)
        cfg1 = SchedulerConfig(**{**config.to_dict(), "resolve_tc2": False})
        alt, _ = resolve_throughput(pool, topology, assignment, cfg1, pl)
        cap = cc3_cap(len(agents), assignment.s, path_length(assignment.s, config.k))

        def hard(nd):  # (CC3, TC1) conflict counts
            cs = detect_conflicts(nd, topology, assignment, topology.mem_capacity, cap=cap)
            return (sum(isinstance(x, StageOveruse) for x in cs), sum(isinstance(x, NodeOveruse) for x in cs))

        ha, hn = hard(alt), hard(node)
        if ha[0] <= hn[0] and ha[1] <= hn[1] and score(alt) < score(node):
            node = alt
        node = _sim_refine(node, score, pl, topology, assignment, cap)
        resolved = not detect_conflicts(node, topology, assignment, topology.mem_capacity, cap=cap)
    return Schedule(config, agents, dict(node.paths), sorted(node.constraints), node.cost, resolved)


def interchangeable_replicas(topology: Topology, assignment: StageAssignment) -> bool:
    """True when, within every stage, the nodes have the same compute times and the same link costs
    to every other node (a uniform box such as one NVSwitch domain): a path's cost then does not
    depend on which replica of a stage it visits."""
    lat, bw = topology.latency_ms, topology.bandwidth_bytes_per_ms
    n = topology.n
    for st in range(assignment.s):
        mem = assignment.stage_nodes(st)
        a = mem[0]
        for b in mem[1:]:
            if topology.compute_fwd_ms[a] != topology.compute_fwd_ms[b]:
                return False
            if topology.compute_bwd_ms(a) != topology.compute_bwd_ms(b):
                return False
            for x in range(n):
                if x in (a, b):
                    continue
                if lat[a][x] != lat[b][x] or bw[a][x] != bw[b][x] or lat[x][a] != lat[x][b] or bw[x][a] != bw[x][b]:
                    return False
            if lat[a][b] != lat[b][a] or bw[a][b] != bw[b][a]:
                return False
    return True


def balance_replicas(sch: Schedule, topology: Topology, assignment: StageAssignment) -> Schedule:
    """Cost-neutral replica re-assignment for interchangeable replicas (B200 extension).

    On a uniform topology A*'s ties go to the lowest node ids, so some replicas carry two paths
    and others none (C2: node 7 never visited) -- harmless in the first-wave plan, but every wave
    repeats it, so per-node work is uneven across the iteration.  Keeping each path's stage
    sequence, the replica of every non-origin visit is re-chosen greedily (agents in id order)
    as the least-loaded one, ties to the lower id.  Applied only when the replicas are
    interchangeable (path costs unchanged) and the re-timed plan keeps CC3 and TC1; otherwise the
    schedule is returned unchanged.  First-wave collisions (TC2) are left to the node queues; the
    caller compares simulated iteration makespans before adopting the result."""
    if not interchangeable_replicas(topology, assignment):
        return sch
    node_stage = assignment.node_stage()
    load = [0] * topology.n
    new_paths = {}
    for a in sorted(sch.paths):
        p = sch.paths[a]
        nodes = [p.nodes[0]]
        for v in p.nodes[1:]:
            st = node_stage[v]
            choice = min(assignment.stage_nodes(st), key=lambda u: (load[u], u))
            nodes.append(choice)
        for v in set(nodes[1:]):
            load[v] += 1
        new_paths[a] = time_fixed_path(a, nodes, topology, assignment, sch.config.msg_bytes)
    cost = max(pp.e2e for pp in new_paths.values())
    if cost > sch.cost_ms + 1e-9:
        return sch
    cand = SearchNode(frozenset(), new_paths, cost)
    if any(not isinstance(c, Collision)
           for c in detect_conflicts(cand, topology, assignment, topology.mem_capacity, k=sch.config.k)):
        return sch
    return Schedule(sch.config, sch.agents, new_paths, sch.constraints, cost, sch.resolved, kind=sch.kind)

