"""The five configurations of BASELINE.json as runnable objects.

Each config bundles the model, stage assignment (explicit sizes — Eq. 1 has no integral
solution on 8 GPUs), the B200 topology the scheduler plans on, the scheduler /
simulator configs and the microbatch shape.  Node compute times for the planner come from the
FLOP model at a nominal sustained rate (``PLAN_TFLOPS``) — they only steer path choice and op
order, and they are frozen here so that the op order (which the executor replays) is a pure
function of the config.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .allocation import StageAssignment
from .model import ModelConfig, layer_split, model_config
from .scheduler import Schedule, SchedulerConfig, balance_replicas, path_length, schedule
from .simulator import SimConfig, simulate
from .topology import Topology, activation_bytes, b200_box

PLAN_TFLOPS = 1000.0   # nominal sustained bf16 rate used only to derive planning times


@dataclass
class RunConfig:
    name: str
    model: ModelConfig
    sizes: list[int]
    k: float
    m: int
    b: int
    T: int
    M: int
    split: list[int] | None = None
    description: str = ""
    kind: str = "skippipe"          # or "full" (dtfm_full sequential pipelines)
    balance_replicas: bool = True   # SkipPipe only: load-balance interchangeable replicas
    swap_every: int = 0             # >0: every swap_every-th agent (ids 1, 1+e, ...) must take one swap
    _cache: dict = field(default_factory=dict, repr=False)

    @property
    def s(self) -> int:
        return len(self.sizes)

    @property
    def assignment(self) -> StageAssignment:
        return StageAssignment.contiguous(self.sizes)

    @property
    def layers(self) -> list[int]:
        return layer_split(self.model, self.s, self.split)

    @property
    def tokens_per_mb(self) -> int:
        return self.b * self.T

    @property
    def msg_bytes(self) -> int:
        return self.model.d * self.T * self.b * 2

    def planning_times(self) -> tuple[list[float], float]:
        """(compute_fwd_ms per node, loss_ms) from the FLOP model at PLAN_TFLOPS."""
        c, n_tok = self.model, self.tokens_per_mb
        stage_of = self.assignment.node_stage()
        fwd = []
        for v in range(sum(self.sizes)):
            fl = self.layers[stage_of[v]] * c.layer_flops_per_token(self.T) * n_tok
            fwd.append(fl / (PLAN_TFLOPS * 1e12) * 1e3)
        loss_ms = 3 * c.head_flops_per_token() * n_tok / (PLAN_TFLOPS * 1e12) * 1e3
        return fwd, loss_ms

    def topology(self) -> Topology:
        fwd, _ = self.planning_times()
        return b200_box(fwd, mem_capacity=self.m)

    def swap_agents(self) -> tuple:
        if self.swap_every <= 0 or self.kind != "skippipe":
            return ()
        n_agents = self.m * self.sizes[0]
        return tuple(range(1, n_agents, self.swap_every))

    def scheduler_config(self) -> SchedulerConfig:
        # sim_select=0: the run configs keep Algorithm 1's plan (SchedulerConfig.sim_select)
        return SchedulerConfig(k=self.k, msg_bytes=float(self.msg_bytes), swap_agents=self.swap_agents(), sim_select=0)

    def swapped_paths(self) -> int:
        """Number of first-wave paths whose stage sequence is reordered (one swap, CC2)."""
        return sum(1 for p in self.schedule().paths.values() if p.swap_count > 0)

    def sim_config(self, record_trace: bool = False) -> SimConfig:
        _, loss_ms = self.planning_times()
        return SimConfig(total_microbatches=self.M, msg_bytes=float(self.msg_bytes), record_trace=record_trace,
                         loss_ms=loss_ms)

    def schedule(self) -> Schedule:
        if "schedule" not in self._cache:
            if self.kind == "full":
                from .baselines import dtfm_full

                self._cache["schedule"] = dtfm_full(self.topology(), self.s, msg_bytes=float(self.msg_bytes),
                                                    assignment=self.assignment)
            elif self.kind == "dtfm_skip":
                from .baselines import dtfm_skip

                self._cache["schedule"] = dtfm_skip(self.topology(), self.assignment, self.scheduler_config())
            elif self.kind == "no_tc2":
                from .baselines import skippipe_no_tc2

                self._cache["schedule"] = skippipe_no_tc2(self.topology(), self.assignment, self.scheduler_config())
            else:
                sch = schedule(self.topology(), self.assignment, self.scheduler_config())
                if self.balance_replicas:
                    # cost-neutral replica re-assignment on the uniform box, kept only when the
                    # simulated iteration does not get slower (scheduler.balance_replicas)
                    bal = balance_replicas(sch, self.topology(), self.assignment)
                    if bal is not sch:
                        sc = self.sim_config()
                        if simulate(bal, self.topology(), sc).iteration_makespan <= \
                                simulate(sch, self.topology(), sc).iteration_makespan:
                            sch = bal
                self._cache["schedule"] = sch
        return self._cache["schedule"]

    def path_len(self) -> int:
        return path_length(self.s, self.k)

    def train_flops(self) -> float:
        """Algorithmic FLOPs of one iteration: 3x forward (fwd + 2x bwd) over every microbatch's
        executed stages + the head, causal attention at half."""
        c = self.model
        sch = self.schedule()
        agents = sorted(a.id for a in sch.agents)
        total = 0.0
        for mb in range(self.M):
            stages = sch.paths[agents[mb % len(agents)]].stages
            per_tok = sum(self.layers[st] for st in stages) * c.layer_flops_per_token(self.T) + c.head_flops_per_token()
            total += 3 * per_tok * self.tokens_per_mb
        return total


# executable baseline variants of a config
VARIANTS = {"-full": "full", "-dtfmskip": "dtfm_skip", "-notc2": "no_tc2"}
# rebalanced layer split: S0 also runs the embedding, the head and the loss of
# every microbatch, so it gets fewer decoder layers; opt-in beside the equal split
REBALANCED = {24: {4: [3, 7, 7, 7]}}


def get_config(name: str, **over) -> RunConfig:
    """C1..C5, plus suffixes (combinable, e.g. "C2-rb-full"): "-m4" memory capacity m = 4
    (8 agents at C2), "-rb" rebalanced layer split (S0 lighter; REBALANCED), "-full" (DT-FM, k=0 disjoint sequential pipelines), "-dtfmskip"
    (DT-FM-skip: topology-blind skip paths, no TC2) and "-notc2" (SkipPipe without the throughput
    phase)."""
    base, suffixes = name, []
    while True:
        suf = next((v for v in list(VARIANTS) + ["-rb", "-m4"] if base.endswith(v)), None)
        if suf is None:
            break
        suffixes.insert(0, suf)
        base = base[: len(base) - len(suf)]
    if base == "C1":
        rc = RunConfig("C1", model_config("llama-50m"), [2, 2, 2, 2], 25, 2, 2, 256, 8,
                       description="tiny LLaMA SkipPipe iteration (4 stages x 2 replicas, 25% skip)")
    elif base == "C2":
        rc = RunConfig("C2", model_config("llama-500m"), [2, 2, 2, 2], 25, 2, 4, 1024, 32,
                       description="LLaMa-500M, 4 stages x 2 replicas, 25% stage skip")
    elif base == "C3":
        # every other agent takes one swap: on the uniform box swaps never lower a path's cost, so
        # without this the scheduler picks none (BASELINE configs[2] names reordered paths)
        rc = RunConfig("C3", model_config("llama-1.5b"), [1] * 8, 25, 8, 1, 4096, 32,
                       description="LLaMa-1.5B, 8 stages x 1, skip + swap (every other path reordered)",
                       swap_every=2)
    elif base == "C4":
        rc = RunConfig("C4", model_config("llama-8b"), [1] * 8, 37.5, 8, 1, 4096, 64,
                       description="LLaMa-8B, 8 stages, 33% skip (l=5 -> effective 37.5%), long queue")
    elif base == "C5":
        rc = RunConfig("C5", model_config("llama-500m"), [2, 2, 2, 2], 50, 2, 4, 1024, 32,
                       description="LLaMa-500M skip sweep point (50%)")
    else:
        raise KeyError(name)
    for suf in suffixes:
        if suf == "-m4":
            # memory capacity m = 4 microbatches per node (TC1): twice the agents in
            # flight -- B200's 180 GB hold them easily -- so fewer pipeline bubbles per wave
            rc.m, rc.name = 4, rc.name + suf
        elif suf == "-rb":
            split = REBALANCED.get(rc.model.n_layers, {}).get(rc.s)
            if split is None:
                raise KeyError(f"{name}: no rebalanced split for {rc.model.n_layers} layers x {rc.s} stages")
            rc.split, rc.name = list(split), rc.name + suf
        elif suf == "-full":
            rc.kind, rc.k, rc.name = "full", 0, rc.name + suf
        else:
            rc.kind, rc.name = VARIANTS[suf], rc.name + suf
    for k_, v in over.items():
        setattr(rc, k_, v)
    return rc
