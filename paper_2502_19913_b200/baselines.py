"""Reference schedulers of the paper's comparison.

* ``dtfm_full``       k = 0 disjoint sequential pipelines, adjacent stages paired by a min-cost
                      assignment — the "full sequential pipeline" that
                      BASELINE.json's metric compares SkipPipe against on the same GPUs.
* ``dtfm_skip``       the scheduler on a unit-cost clone, TC2 off (Appendix B).
* ``skippipe_no_tc2`` the scheduler with TC2 resolution off.
* ``compensate``      DT-FM* node-count compensation.
"""

from __future__ import annotations

import numpy as np
from scipy.optimize import linear_sum_assignment

from .allocation import GAConfig, StageAssignment, cluster_nodes, order_stages
from .errors import ValidationError
from .scheduler import Schedule, SchedulerConfig, make_agents, schedule, time_fixed_path
from .topology import Topology, comm_matrix


def dtfm_full(topology: Topology, s: int, *, msg_bytes: float, assignment: StageAssignment | None = None,
              ga_config: GAConfig | None = None) -> Schedule:
    if assignment is None:
        if topology.n % s:
            raise ValidationError(f"dtfm_full needs n divisible by s (n={topology.n}, s={s})")
        members = cluster_nodes(topology, [topology.n // s] * s, ga_config)
        assignment = order_stages(topology, members, msg_bytes)
    if len(set(assignment.sizes)) != 1:
        raise ValidationError(f"dtfm_full needs equal stage sizes, got {assignment.sizes}")
    cm = comm_matrix(topology, msg_bytes)
    chains = [[v] for v in assignment.stage_nodes(0)]
    for st in range(1, assignment.s):
        nxt = assignment.stage_nodes(st)
        cost = np.array([[cm[c[-1], v] for v in nxt] for c in chains])
        rows, cols = linear_sum_assignment(cost)
        for r, c in zip(rows, cols):
            chains[r].append(nxt[c])
    by_origin = {c[0]: c for c in chains}
    agents = make_agents(assignment, topology.mem_capacity)
    paths = {a.id: time_fixed_path(a.id, by_origin[a.origin], topology, assignment, msg_bytes) for a in agents}
    cfg = SchedulerConfig(k=0, msg_bytes=msg_bytes)
    return Schedule(cfg, agents, paths, [], max(p.e2e for p in paths.values()), True, kind="DtfmFull")


def unit_cost_clone(topology: Topology) -> Topology:
    n = topology.n
    lat = np.ones((n, n))
    bw = np.full((n, n), 1e30)
    np.fill_diagonal(lat, 0.0)
    np.fill_diagonal(bw, 1.0)
    return Topology(n=n, latency_ms=lat, bandwidth_bytes_per_ms=bw, compute_fwd_ms=np.ones(n), bwd_ratio=1.0,
                    mem_capacity=topology.mem_capacity)


def dtfm_skip(topology: Topology, assignment: StageAssignment, config: SchedulerConfig) -> Schedule:
    cfg = SchedulerConfig(**{**config.to_dict(), "resolve_tc2": False})
    sch = schedule(unit_cost_clone(topology), assignment, cfg)
    # re-time the chosen node sequences on the true topology
    paths = {a: time_fixed_path(a, list(p.nodes), topology, assignment, config.msg_bytes) for a, p in sch.paths.items()}
    return Schedule(cfg, sch.agents, paths, sch.constraints, max(p.e2e for p in paths.values()), sch.resolved,
                    kind="DtfmSkip")


def skippipe_no_tc2(topology: Topology, assignment: StageAssignment, config: SchedulerConfig) -> Schedule:
    cfg = SchedulerConfig(**{**config.to_dict(), "resolve_tc2": False})
    sch = schedule(topology, assignment, cfg)
    sch.kind = "SkipPipeNoTc2"
    return sch


def compensate(time_ms: float, nodes_used: int, nodes_total: int) -> float:
    """time × used/total — DT-FM* credit for unused nodes (§4.1)."""
    if nodes_used <= 0 or nodes_total <= 0:
        raise ValidationError("compensate needs positive node counts")
    if nodes_used > nodes_total:
        raise ValidationError(f"nodes_used={nodes_used} exceeds nodes_total={nodes_total}")
    return time_ms * nodes_used / nodes_total
