"""Deterministic discrete-event simulator of a schedule.

Each node runs one op at a time; arrivals queue; backward-class work (B and the loss op L) is
picked before forward work (1F1B); a node holding m active microbatches defers new
forward work until a backward completes (TC1 memory); links never collide
(full duplex); when a microbatch's backward reaches its origin the next wave
launches on the same path.  Queue order within a class: FIFO by arrival,
then wave, then agent id.

Beyond the spec, every executed compute op is returned as an :class:`Op` with the memory slot it
occupies on its node.  The B200 executor replays exactly this per-node order (the north star's
"per-node op order bit-exact"), so the simulator is the single source of truth for op order.

The loss op ``L`` (final norm, de-embedding and cross-entropy at the origin on the forward
return) is absent from the spec's cost model; ``SimConfig.loss_ms`` gives it a
duration.  With the default 0 it occupies no node time and the spec's arithmetic is unchanged
(SURVEY.md §7 H5).
"""

from __future__ import annotations

import csv
import heapq
import io
import json
from dataclasses import dataclass, field

from .errors import ValidationError
from .scheduler import Schedule
from .topology import Topology, comm_matrix

F, L, B = "F", "L", "B"
_DIRECTION = {F: "fwd", L: "loss", B: "bwd"}


@dataclass(frozen=True)
class SimConfig:
    total_microbatches: int
    msg_bytes: float
    record_trace: bool = False
    loss_ms: float = 0.0
    bwd_msg_bytes: float | None = None   # backward messages default to msg_bytes
    # B200 extension (not in SPEC): node -> device.  Logical nodes placed on one GPU share its
    # compute: a device runs one op at a time, picking B / L before F and then the earliest ready
    # op over all its nodes.  None = one device per node (the spec's model).
    device_of: tuple | None = None

    def __post_init__(self):
        if self.total_microbatches < 1:
            raise ValidationError("total_microbatches must be >= 1")
        if not self.msg_bytes > 0:
            raise ValidationError("msg_bytes must be positive")
        if self.loss_ms < 0:
            raise ValidationError("loss_ms must be >= 0")


@dataclass(frozen=True)
class Op:
    """One executed compute op.  ``pos`` is the index of ``node`` in the microbatch's path
    (origin = 0); ``slot`` is the node-local activation slot (0..m-1) the microbatch holds."""

    kind: str
    node: int
    agent: int
    wave: int
    mb: int
    pos: int
    stage: int
    ready: float
    start: float
    end: float
    slot: int


@dataclass
class SimReport:
    iteration_makespan: float
    microbatch_e2e: list[float]
    total_collision_wait: float
    node_busy: list[float]
    node_idle: list[float]
    ops: list[Op]
    cap_overrides: int = 0
    trace: list[tuple] | None = None

    def node_order(self) -> dict[int, list[tuple[str, int, int]]]:
        """node -> [(kind, agent, wave), ...] in execution order."""
        out: dict[int, list] = {}
        for op in self.ops:
            out.setdefault(op.node, []).append((op.kind, op.agent, op.wave))
        return out

    def to_dict(self) -> dict:
        return {
            "iteration_makespan": self.iteration_makespan,
            "microbatch_e2e": self.microbatch_e2e,
            "total_collision_wait": self.total_collision_wait,
            "node_busy": self.node_busy,
            "node_idle": self.node_idle,
            "cap_overrides": self.cap_overrides,
        }

    def dumps(self) -> str:
        return json.dumps(self.to_dict(), indent=2, sort_keys=True) + "\n"

    def trace_csv(self) -> str:
        if self.trace is None:
            raise ValidationError("report was recorded without a trace; rerun with record_trace=True (--trace)")
        buf = io.StringIO()
        w = csv.writer(buf, lineterminator="\n")
        w.writerow(["time_ms", "node", "event", "agent", "wave", "direction"])
        for row in self.trace:
            w.writerow([repr(float(row[0])), *row[1:]])
        return buf.getvalue()


def simulate(schedule: Schedule, topology: Topology, sim_config: SimConfig) -> SimReport:
    """Run M = total_microbatches microbatches over the schedule's first-wave paths."""
    agents = sorted(a.id for a in schedule.agents)
    index_of = {a: i for i, a in enumerate(agents)}
    n_agents = len(agents)
    M = sim_config.total_microbatches
    if M % n_agents:
        raise ValidationError(f"total_microbatches={M} is not divisible by the {n_agents} agents (one wave = |P|)")
    waves = M // n_agents
    paths = {a: schedule.paths[a].nodes for a in agents}
    stage_of = {a: schedule.paths[a].stages for a in agents}
    for a, nodes in paths.items():
        for v in nodes:
            if not (0 <= v < topology.n):
                raise ValidationError(f"path of agent {a} references unknown node {v}", row=a)
    n, m = topology.n, topology.mem_capacity
    fwd = topology.compute_fwd_ms
    cm_f = comm_matrix(topology, sim_config.msg_bytes)
    cm_b = comm_matrix(topology, sim_config.bwd_msg_bytes or sim_config.msg_bytes)
    loss_ms = float(sim_config.loss_ms)

    dev = list(sim_config.device_of) if sim_config.device_of is not None else list(range(n))
    if len(dev) != n:
        raise ValidationError(f"device_of has {len(dev)} entries for {n} nodes")
    dev_nodes: dict[int, list[int]] = {}
    for v in range(n):
        dev_nodes.setdefault(dev[v], []).append(v)
    running = {d: False for d in dev_nodes}  # per device
    active = [0] * n
    free_slots = [list(range(m)) for _ in range(n)]
    slot_of: dict[tuple[int, int], int] = {}     # (mb, node) -> slot
    queue_b: list[list] = [[] for _ in range(n)]  # entries (ready, wave, agent, kind, pos)
    queue_f: list[list] = [[] for _ in range(n)]
    busy = [0.0] * n
    ops: list[Op] = []
    trace: list | None = [] if sim_config.record_trace else None
    e2e = [0.0] * M
    launch = [0.0] * M
    stats = {"wait": 0.0, "overrides": 0}

    events: list = []   # (time, order, seq, payload); completions (order 0) before arrivals (order 1)
    counter = [0]

    def push(t, order, payload):
        heapq.heappush(events, (float(t), order, counter[0], payload))
        counter[0] += 1

    def mb_id(agent, wave):
        return wave * n_agents + index_of[agent]

    def record(kind, v, agent, wave, pos, ready, t0, t1, slot):
        ops.append(Op(kind, v, agent, wave, mb_id(agent, wave), pos, stage_of[agent][pos], ready, t0, t1, slot))
        if trace is not None:
            trace.append((t0, v, "start", agent, wave, _DIRECTION[kind]))
            trace.append((t1, v, "end", agent, wave, _DIRECTION[kind]))

    def start(v, t, entry):
        ready, wave, agent, kind, pos = entry
        mb = mb_id(agent, wave)
        if kind == F:
            slot = free_slots[v].pop(0) if free_slots[v] else -1   # -1 only after a cap override
            slot_of[(mb, v)] = slot
            active[v] += 1
            dur = float(fwd[v])
        else:
            slot = slot_of[(mb, v)]
            dur = topology.compute_bwd_ms(v) if kind == B else loss_ms
        stats["wait"] += t - ready
        running[dev[v]] = True
        busy[v] += dur
        record(kind, v, agent, wave, pos, ready, t, t + dur, slot)
        push(t + dur, 0, ("done", v, kind, agent, wave, pos))

    def complete(t, v, kind, agent, wave, pos):
        """Work that follows a finished op: the next hop's arrival, slot release, next wave."""
        nodes = paths[agent]
        last = len(nodes) - 1
        if kind == F:
            if pos < last:
                nxt = nodes[pos + 1]
                push(t + cm_f[v, nxt], 1, ("arrive", nxt, F, agent, wave, pos + 1))
            else:
                o = nodes[0]
                push(t + (cm_f[v, o] if v != o else 0.0), 1, ("arrive", o, L, agent, wave, 0))
        elif kind == L:
            tgt = nodes[last]
            push(t + (cm_b[v, tgt] if v != tgt else 0.0), 1, ("arrive", tgt, B, agent, wave, last))
        else:
            mb = mb_id(agent, wave)
            active[v] -= 1
            slot = slot_of.pop((mb, v))
            if slot >= 0:
                free_slots[v].append(slot)
                free_slots[v].sort()
            if pos > 0:
                prev = nodes[pos - 1]
                push(t + cm_b[v, prev], 1, ("arrive", prev, B, agent, wave, pos - 1))
            else:
                e2e[mb] = t - launch[mb]
                if wave + 1 < waves:
                    launch[mb_id(agent, wave + 1)] = t
                    push(t, 1, ("arrive", nodes[0], F, agent, wave + 1, 0))

    for a in agents:
        push(0.0, 1, ("arrive", paths[a][0], F, a, 0, 0))

    while events or any(queue_f) or any(queue_b):
        if events:
            t = events[0][0]
            while events and events[0][0] == t:
                _, _, _, (what, v, kind, agent, wave, pos) = heapq.heappop(events)
                if what == "done":
                    running[dev[v]] = False
                    complete(t, v, kind, agent, wave, pos)
                elif kind == L and loss_ms == 0.0:
                    # the spec's cost model has no loss compute: the return passes straight through
                    record(L, v, agent, wave, 0, t, t, t, slot_of[(mb_id(agent, wave), v)])
                    complete(t, v, L, agent, wave, pos)
                else:
                    (queue_f if kind == F else queue_b)[v].append((t, wave, agent, kind, pos))
        else:
            # only forwards deferred by the memory cap remain and nothing can free a slot:
            # admit the earliest one over the cap so that any schedule stays executable
            v = min((v for v in range(n) if queue_f[v]), key=lambda v: (min(queue_f[v]), v))
            queue_f[v].sort()
            stats["overrides"] += 1
            start(v, t, queue_f[v].pop(0))
            continue
        for d in sorted(dev_nodes):
            if running[d]:
                continue
            nodes_d = dev_nodes[d]
            cand = [(min(queue_b[v]), v) for v in nodes_d if queue_b[v]]
            qs = queue_b
            if not cand:
                cand = [(min(queue_f[v]), v) for v in nodes_d if queue_f[v] and active[v] < m]
                qs = queue_f
            if cand:
                entry, v = min(cand)
                qs[v].remove(entry)
                start(v, t, entry)

    makespan = max((op.end for op in ops), default=0.0)
    return SimReport(
        iteration_makespan=makespan,
        microbatch_e2e=e2e,
        total_collision_wait=stats["wait"],
        node_busy=busy,
        node_idle=[makespan - b for b in busy],
        ops=ops,
        cap_overrides=stats["overrides"],
        trace=trace,
    )


def replay_makespan(ops, schedule: Schedule, topology: Topology, sim_config: SimConfig, device_of) -> float:
    """Makespan of executing ``ops`` in exactly this order on devices (node -> device_of[node]):
    each device runs its ops one at a time in list order, an op starts when its device is free and
    its input has arrived (the previous op of its path plus the hop).  This is how the executor
    replays an op list on one stream per GPU, so it scores candidate orders."""
    cm_f = comm_matrix(topology, sim_config.msg_bytes)
    cm_b = comm_matrix(topology, sim_config.bwd_msg_bytes or sim_config.msg_bytes)
    paths = {a: schedule.paths[a].nodes for a in schedule.paths}
    end: dict = {}
    free: dict = {}
    for op in ops:
        a, w, pos, v = op.agent, op.wave, op.pos, op.node
        nodes = paths[a]
        last = len(nodes) - 1
        if op.kind == F:
            if pos > 0:
                r = end[(F, a, w, pos - 1)] + cm_f[nodes[pos - 1], v]
            else:
                r = end[(B, a, w - 1, 0)] if w > 0 else 0.0
            dur = float(topology.compute_fwd_ms[v])
        elif op.kind == L:
            r = end[(F, a, w, last)] + (cm_f[nodes[last], v] if nodes[last] != v else 0.0)
            dur = float(sim_config.loss_ms)
        else:
            if pos == last:
                r = end[(L, a, w, 0)] + (cm_b[nodes[0], v] if nodes[0] != v else 0.0)
            else:
                r = end[(B, a, w, pos + 1)] + cm_b[nodes[pos + 1], v]
            dur = topology.compute_bwd_ms(v)
        d = device_of[v]
        t0 = max(free.get(d, 0.0), r)
        end[(op.kind, a, w, pos)] = free[d] = t0 + dur
    return max(end.values(), default=0.0)


def compare(schedules: dict, topology: Topology, sim_config: SimConfig) -> list[dict]:
    """Per-schedule report plus speed-up of the first (by name) over each."""
    names = sorted(schedules)
    reps = {nm: simulate(schedules[nm], topology, sim_config) for nm in names}
    base = reps[names[0]].iteration_makespan if names else 0.0
    return [{"name": nm, "makespan_ms": reps[nm].iteration_makespan,
             "speedup_vs_first": (base / reps[nm].iteration_makespan) if reps[nm].iteration_makespan else 1.0,
             "collision_wait_ms": reps[nm].total_collision_wait} for nm in names]
