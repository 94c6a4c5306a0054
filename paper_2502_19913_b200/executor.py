"""B200 partial-pipeline training executor: the drop-in for ``simulate`` that runs
the schedule for real.

``execute(schedule, topology, sim_config, model_cfg, placement, tokens)`` takes the same
schedule / topology / sim_config as the reference's simulator plus the model, a placement of
logical nodes onto GPUs and the synthetic tokens, and returns an :class:`ExecReport` that has
the SimReport fields measured on the GPU plus the losses.  ``Trainer`` is the reusable object
behind it (``bench.py`` and the tests drive ``Trainer.step``).

Execution model:
* The simulator's op list (F / L / B per node, in start-time order, with the node-local memory
  slot of every microbatch) is the program.  The executor replays it in that global order, so
  the per-node op order equals the simulated one by construction, and records what it issued
  (``ExecReport.node_order``) so the tests can check it.
* Every (node, slot, op-kind) is one CUDA graph captured once at setup over fixed buffers:
  ~50 (F) / ~100 (B) kernels per 6-layer stage replay with one launch.  Per-microbatch inputs
  (token ids, targets, embedding-backward segments) are staged into the slot's buffers by small
  async copies before the replay.
* A path hop copies the producer's output into the consumer node's slot buffer with
  ``spx_hop`` (NVLink peer copy across GPUs, D2D on one GPU).
* Replicas of a stage that live on the same GPU share one parameter set (their gradients would
  be summed by the replica all-reduce anyway); across GPUs the replica sets are all-reduced with
  NCCL (``Trainer.sync_grads``).  Then global-norm clip and AdamW run on the device without a
  host sync; the loss is read back once per iteration.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import torch

from . import native
from .errors import ValidationError
from .model import (ModelConfig, StageLayout, init_params, layer_split, pack_stage, rope_cos_sin, stage_layout,
                    unpack_stage)
from .scheduler import Schedule
from .simulator import B, F, L, SimConfig, SimReport, simulate
from .topology import Topology

BF16 = torch.bfloat16
F32 = torch.float32


@dataclass(frozen=True)
class OptimConfig:
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1
    max_grad_norm: float = 1.0


@dataclass
class ExecReport:
    """SimReport fields measured on the GPU, plus training outputs."""

    iteration_makespan: float            # ms, first op issue -> optimizer done (CUDA events)
    microbatch_e2e: list[float]          # ms, F at origin start -> B at origin end
    total_collision_wait: float          # ms, sum over ops of (start - ready) on the device timeline
    node_busy: list[float]
    node_idle: list[float]
    loss: float
    mb_loss: list[float]
    grad_norm: float
    node_order: dict = field(default_factory=dict)   # node -> [(kind, agent, wave)] as executed
    trace: list | None = None


# ---------------------------------------------------------------------------------------
# device-side state
# ---------------------------------------------------------------------------------------
class ParamSet:
    """One stage's parameters on one device: flat fp32 master / bf16 copy / grad / Adam moments."""

    def __init__(self, cfg: ModelConfig, lay: StageLayout, flat32_cpu: torch.Tensor, device):
        self.cfg, self.lay, self.device = cfg, lay, device
        self.p32 = flat32_cpu.to(device)
        self.pbf = self.p32.to(BF16)
        self.g = torch.zeros_like(self.p32)
        self.m = torch.zeros_like(self.p32)
        self.v = torch.zeros_like(self.p32)

    def w(self, name):
        return self.lay.view(self.pbf, name)

    def gv(self, name):
        return self.lay.view(self.g, name)


class LayerActs:
    """Saved activations of one decoder layer for one (node, slot)."""

    def __init__(self, cfg: ModelConfig, n: int, b: int, T: int, device):
        d, f = cfg.d, cfg.ffn
        e = dict(dtype=BF16, device=device)
        self.xn1 = torch.empty(n, d, **e)
        self.rstd1 = torch.empty(n, dtype=F32, device=device)
        self.qkv = torch.empty(n, cfg.qkv_dim, **e)
        self.o = torch.empty(n, cfg.n_heads * cfg.head_dim, **e)
        self.lse = torch.empty(b, cfg.n_heads, T, dtype=F32, device=device)
        self.xmid = torch.empty(n, d, **e)
        self.xn2 = torch.empty(n, d, **e)
        self.rstd2 = torch.empty(n, dtype=F32, device=device)
        self.gu = torch.empty(n, 2 * f, **e)
        self.h = torch.empty(n, f, **e)


class SlotBuffers:
    """Everything a microbatch keeps on a node while it holds one of the node's m slots."""

    def __init__(self, cfg: ModelConfig, n_layers: int, origin: bool, n: int, b: int, T: int, device):
        e = dict(dtype=BF16, device=device)
        self.xs = [torch.empty(n, cfg.d, **e) for _ in range(n_layers + 1)]  # residual stream
        self.layers = [LayerActs(cfg, n, b, T, device) for _ in range(n_layers)]
        self.gin = torch.empty(n, cfg.d, **e)           # gradient w.r.t. this node's output
        if origin:
            self.ids = torch.zeros(n, dtype=torch.int32, device=device)
            self.targets = torch.zeros(n, dtype=torch.int32, device=device)
            self.perm = torch.zeros(n, dtype=torch.int32, device=device)
            self.seg_start = torch.zeros(n + 1, dtype=torch.int32, device=device)
            self.seg_id = torch.zeros(n, dtype=torch.int32, device=device)
            self.n_seg = torch.zeros(1, dtype=torch.int32, device=device)
            self.ret = torch.empty(n, cfg.d, **e)       # activation returned to the origin (L input)
            self.loss = torch.zeros(1, dtype=F32, device=device)


class Scratch:
    """Per-device scratch shared by all ops of that device (ops are serialised on its stream)."""

    def __init__(self, cfg: ModelConfig, n: int, b: int, T: int, device, with_head: bool):
        d, f = cfg.d, cfg.ffn
        e = dict(dtype=BF16, device=device)
        self.dx = [torch.empty(n, d, **e) for _ in range(2)]
        self.dxm = torch.empty(n, d, **e)
        self.dxn = torch.empty(n, d, **e)
        self.dh = torch.empty(n, f, **e)
        self.dgu = torch.empty(n, 2 * f, **e)
        self.do = torch.empty(n, cfg.n_heads * cfg.head_dim, **e)
        self.dqkv = torch.empty(n, cfg.qkv_dim, **e)
        self.delta = torch.empty(b, cfg.n_heads, T, dtype=F32, device=device)
        self.rms_ws = torch.empty(native.rmsnorm_ws_floats(d), dtype=F32, device=device)
        self.rope = rope_cos_sin(T, cfg.head_dim, cfg.rope_theta).to(device)
        if with_head:
            self.xf = torch.empty(n, d, **e)
            self.rstdf = torch.empty(n, dtype=F32, device=device)
            self.logits = torch.empty(n, cfg.vocab, **e)
            self.row_loss = torch.empty(n, dtype=F32, device=device)
            self.dxf = torch.empty(n, d, **e)
            self.dret = torch.empty(n, d, **e)


# ---------------------------------------------------------------------------------------
# stage programs (sequences of libspx calls on one stream)
# ---------------------------------------------------------------------------------------
class StageProgram:
    def __init__(self, cfg: ModelConfig, n: int, b: int, T: int, M: int):
        self.cfg, self.n, self.b, self.T, self.M = cfg, n, b, T, M
        self.scale = 1.0 / math.sqrt(cfg.head_dim)

    # ---- one decoder layer ----
    def layer_fwd(self, ps: ParamSet, i: int, x, a: LayerActs, y, sc: Scratch, s):
        c, n = self.cfg, self.n
        d, f, qd, hd = c.d, c.ffn, c.qkv_dim, c.head_dim
        od = c.n_heads * hd
        native.rmsnorm_fwd(x, ps.w(f"l{i}.attn_norm"), a.xn1, a.rstd1, rows=n, d=d, eps=c.eps, stream=s)
        native.gemm(a.xn1, ps.w(f"l{i}.wqkv"), a.qkv, M=n, N=qd, K=d, lda=d, ldb=d, ldc=qd, stream=s)
        native.rope(a.qkv, sc.rope, rows=n, T=self.T, n_heads=c.n_heads + c.n_kv_heads, hd=hd, ld=qd, stream=s)
        native.attn_fwd(a.qkv, a.o, a.lse, B=self.b, T=self.T, H=c.n_heads, Hkv=c.n_kv_heads, hd=hd, ld_qkv=qd,
                        ld_o=od, scale=self.scale, stream=s)
        native.gemm(a.o, ps.w(f"l{i}.wo"), a.xmid, M=n, N=d, K=od, lda=od, ldb=od, ldc=d,
                    epilogue=native.EPI_BF16_RESID, R=x, stream=s)
        native.rmsnorm_fwd(a.xmid, ps.w(f"l{i}.mlp_norm"), a.xn2, a.rstd2, rows=n, d=d, eps=c.eps, stream=s)
        native.gemm(a.xn2, ps.w(f"l{i}.wgu"), a.h, M=n, N=2 * f, K=d, lda=d, ldb=d, ldc=f,
                    epilogue=native.EPI_SWIGLU, C2=a.gu, ldc2=2 * f, stream=s)
        native.gemm(a.h, ps.w(f"l{i}.wdown"), y, M=n, N=d, K=f, lda=f, ldb=f, ldc=d,
                    epilogue=native.EPI_BF16_RESID, R=a.xmid, stream=s)

    def layer_bwd(self, ps: ParamSet, i: int, x, a: LayerActs, dy, dx, sc: Scratch, s):
        """dy: grad of the layer output; dx: grad of the layer input (may not alias dy)."""
        c, n = self.cfg, self.n
        d, f, qd, hd = c.d, c.ffn, c.qkv_dim, c.head_dim
        od = c.n_heads * hd
        F32E = native.EPI_F32
        # MLP
        native.gemm(dy, ps.w(f"l{i}.wdown"), sc.dh, M=n, N=f, K=d, lda=d, ldb=f, ldc=f, b_mn=True, stream=s)
        native.gemm(dy, a.h, ps.gv(f"l{i}.wdown"), M=d, N=f, K=n, lda=d, ldb=f, ldc=f, a_mn=True, b_mn=True,
                    epilogue=F32E, beta=1.0, stream=s)
        native.swiglu_bwd(a.gu, sc.dh, sc.dgu, rows=n, F=f, stream=s)
        native.gemm(sc.dgu, ps.w(f"l{i}.wgu"), sc.dxn, M=n, N=d, K=2 * f, lda=2 * f, ldb=d, ldc=d, b_mn=True,
                    stream=s)
        native.gemm(sc.dgu, a.xn2, ps.gv(f"l{i}.wgu"), M=2 * f, N=d, K=n, lda=2 * f, ldb=d, ldc=d, a_mn=True,
                    b_mn=True, epilogue=F32E, beta=1.0, stream=s)
        native.rmsnorm_bwd(a.xmid, ps.w(f"l{i}.mlp_norm"), a.rstd2, sc.dxn, dy, sc.dxm, ps.gv(f"l{i}.mlp_norm"),
                           sc.rms_ws, rows=n, d=d, stream=s)
        # attention
        native.gemm(sc.dxm, ps.w(f"l{i}.wo"), sc.do, M=n, N=od, K=d, lda=d, ldb=od, ldc=od, b_mn=True, stream=s)
        native.gemm(sc.dxm, a.o, ps.gv(f"l{i}.wo"), M=d, N=od, K=n, lda=d, ldb=od, ldc=od, a_mn=True, b_mn=True,
                    epilogue=F32E, beta=1.0, stream=s)
        native.attn_bwd(a.qkv, a.o, sc.do, a.lse, sc.delta, sc.dqkv, B=self.b, T=self.T, H=c.n_heads,
                        Hkv=c.n_kv_heads, hd=hd, ld_qkv=qd, ld_o=od, scale=self.scale, stream=s)
        native.rope(sc.dqkv, sc.rope, rows=n, T=self.T, n_heads=c.n_heads + c.n_kv_heads, hd=hd, ld=qd, inverse=True,
                    stream=s)
        native.gemm(sc.dqkv, ps.w(f"l{i}.wqkv"), sc.dxn, M=n, N=d, K=qd, lda=qd, ldb=d, ldc=d, b_mn=True, stream=s)
        native.gemm(sc.dqkv, a.xn1, ps.gv(f"l{i}.wqkv"), M=qd, N=d, K=n, lda=qd, ldb=d, ldc=d, a_mn=True, b_mn=True,
                    epilogue=F32E, beta=1.0, stream=s)
        native.rmsnorm_bwd(x, ps.w(f"l{i}.attn_norm"), a.rstd1, sc.dxn, sc.dxm, dx, ps.gv(f"l{i}.attn_norm"),
                           sc.rms_ws, rows=n, d=d, stream=s)

    # ---- node ops ----
    def fwd(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, origin: bool, s):
        if origin:
            native.embed_fwd(sb.ids, ps.w("embed"), sb.xs[0], n=self.n, d=self.cfg.d, stream=s)
        for i, a in enumerate(sb.layers):
            self.layer_fwd(ps, i, sb.xs[i], a, sb.xs[i + 1], sc, s)

    def bwd(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, origin: bool, s):
        """Returns the buffer holding the gradient w.r.t. the node's input."""
        dy = sb.gin
        k = 0
        for i in reversed(range(len(sb.layers))):
            dx = sc.dx[k]
            self.layer_bwd(ps, i, sb.xs[i], sb.layers[i], dy, dx, sc, s)
            dy, k = dx, k ^ 1
        if origin:
            native.embed_bwd(sb.perm, sb.seg_start, sb.seg_id, sb.n_seg, self.n, dy, ps.gv("embed"), d=self.cfg.d,
                             stream=s)
        return dy

    def loss(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, s):
        """Final norm, de-embedding, cross-entropy fwd+bwd at the origin."""
        c, n = self.cfg, self.n
        d, V = c.d, c.vocab
        native.rmsnorm_fwd(sb.ret, ps.w("final_norm"), sc.xf, sc.rstdf, rows=n, d=d, eps=c.eps, stream=s)
        native.gemm(sc.xf, ps.w("head"), sc.logits, M=n, N=V, K=d, lda=d, ldb=d, ldc=V, stream=s)
        native.xent_fwd_bwd(sc.logits, sb.targets, sc.row_loss, n=n, V=V, ld=V, scale=1.0 / (n * self.M), stream=s)
        native.sum_f32(sc.row_loss, n, sb.loss, scale=1.0 / n, stream=s)
        native.gemm(sc.logits, ps.w("head"), sc.dxf, M=n, N=d, K=V, lda=V, ldb=d, ldc=d, b_mn=True, stream=s)
        native.gemm(sc.logits, sc.xf, ps.gv("head"), M=V, N=d, K=n, lda=V, ldb=d, ldc=d, a_mn=True, b_mn=True,
                    epilogue=native.EPI_F32, beta=1.0, stream=s)
        native.rmsnorm_bwd(sb.ret, ps.w("final_norm"), sc.rstdf, sc.dxf, None, sc.dret, ps.gv("final_norm"),
                           sc.rms_ws, rows=n, d=d, stream=s)
        return sc.dret


# ---------------------------------------------------------------------------------------
# the trainer
# ---------------------------------------------------------------------------------------
def default_placement(n_nodes: int, n_gpus: int) -> list[int]:
    """Logical node i -> GPU i mod n_gpus (contiguous stage numbering makes this spread each
    stage's replicas over different GPUs when n_gpus divides the replica count)."""
    return [i % n_gpus for i in range(n_nodes)]


class Trainer:
    """Holds weights, optimizer state, activation slots and captured graphs for one config.

    Single process; all logical nodes placed on this process's devices.  (The multi-process
    NVLink/NCCL path is ``dist_trainer.DistTrainer``.)"""

    def __init__(self, schedule: Schedule, topology: Topology, sim_config: SimConfig, cfg: ModelConfig,
                 assignment, *, b: int, T: int | None = None, split: list[int] | None = None,
                 placement: list[int] | None = None, seed: int = 0, optim: OptimConfig | None = None,
                 use_graphs: bool = True, params: list | None = None):
        if not torch.cuda.is_available():
            raise native.NativeError("the executor needs a CUDA device (there is no CPU fallback)")
        native.load()
        self.schedule, self.topology, self.sim_config = schedule, topology, sim_config
        self.cfg, self.assignment = cfg, assignment
        self.T = T or cfg.context
        self.b = b
        self.n = b * self.T
        self.M = sim_config.total_microbatches
        self.split = layer_split(cfg, assignment.s, split)
        self.optim = optim or OptimConfig()
        self.node_stage = assignment.node_stage()
        self.placement = placement or [0] * topology.n
        if len(self.placement) != topology.n:
            raise ValidationError(f"placement has {len(self.placement)} entries for {topology.n} nodes")
        self.devices = sorted(set(self.placement))
        self.report: SimReport = simulate(schedule, topology, sim_config)
        self.ops = self.report.ops
        self.step_count = 0
        self.use_graphs = use_graphs
        self.agents = sorted(a.id for a in schedule.agents)
        self.paths = {a: schedule.paths[a].nodes for a in self.agents}

        # parameter sets: one per (stage, device)
        canon = params if params is not None else init_params(cfg, self.split, seed)
        self.layouts = [stage_layout(cfg, st, self.split) for st in range(assignment.s)]
        self.psets: dict[tuple[int, int], ParamSet] = {}
        for v in range(topology.n):
            st, dev = self.node_stage[v], self.placement[v]
            if (st, dev) not in self.psets:
                flat = pack_stage(cfg, self.layouts[st], canon[st])
                self.psets[(st, dev)] = ParamSet(cfg, self.layouts[st], flat, torch.device("cuda", dev))
        # activation slots per node
        m = topology.mem_capacity
        self.slots: dict[tuple[int, int], SlotBuffers] = {}
        for v in range(topology.n):
            dev = torch.device("cuda", self.placement[v])
            for j in range(m):
                self.slots[(v, j)] = SlotBuffers(cfg, self.split[self.node_stage[v]], self.node_stage[v] == 0,
                                                 self.n, b, self.T, dev)
        self.scratch = {d: Scratch(cfg, self.n, b, self.T, torch.device("cuda", d),
                                   with_head=any(self.node_stage[v] == 0 and self.placement[v] == d
                                                 for v in range(topology.n)))
                        for d in self.devices}
        self.streams = {d: torch.cuda.Stream(device=d) for d in self.devices}
        self.prog = StageProgram(cfg, self.n, b, self.T, self.M)
        self.mb_loss = torch.zeros(self.M, dtype=F32, device=torch.device("cuda", self.devices[0]))
        self._slot_of = {(op.mb, op.node): op.slot for op in self.ops if op.kind == F}
        self._graphs: dict = {}
        self._graph_launches: dict = {}
        self._graph_gemms: dict = {}
        self._opt_launches = 0
        self._bwd_out: dict = {}
        self._sumsq = {d: torch.zeros(len(self.psets), dtype=F32, device=torch.device("cuda", d)) for d in self.devices}
        self._sumsq_ws = {d: torch.empty(native.sumsq_ws_floats(), dtype=F32, device=torch.device("cuda", d))
                          for d in self.devices}
        self._clip = {d: torch.ones(1, dtype=F32, device=torch.device("cuda", d)) for d in self.devices}
        self._norm = {d: torch.zeros(1, dtype=F32, device=torch.device("cuda", d)) for d in self.devices}
        for a in self.devices:
            for c in self.devices:
                if a != c:
                    native.enable_peer_access(a, c)
        if use_graphs:
            self._capture_all()

    # ---- graph capture ----
    def _run_op(self, kind: str, v: int, slot: int, s):
        dev = self.placement[v]
        ps = self.psets[(self.node_stage[v], dev)]
        sb = self.slots[(v, slot)]
        sc = self.scratch[dev]
        origin = self.node_stage[v] == 0
        if kind == F:
            self.prog.fwd(ps, sb, sc, origin, s)
            return sb.xs[-1]
        if kind == L:
            return self.prog.loss(ps, sb, sc, s)
        return self.prog.bwd(ps, sb, sc, origin, s)

    def _capture_all(self):
        keys = sorted({(op.kind, op.node, op.slot) for op in self.ops})
        for kind, v, slot in keys:
            dev = self.placement[v]
            with torch.cuda.device(dev):
                s = self.streams[dev]
                g = torch.cuda.CUDAGraph()
                s.wait_stream(torch.cuda.current_stream())
                n0 = native.launches()
                native.take_gemm_log()
                with torch.cuda.graph(g, stream=s):
                    out = self._run_op(kind, v, slot, torch.cuda.current_stream())
                self._graph_launches[(kind, v, slot)] = native.launches() - n0
                self._graph_gemms[(kind, v, slot)] = native.take_gemm_log()
                self._graphs[(kind, v, slot)] = g
                self._bwd_out[(kind, v, slot)] = out
        torch.cuda.synchronize()

    # ---- one iteration ----
    def _stage_inputs(self, tokens: torch.Tensor):
        """Pinned host copies of ids / targets / embedding-backward segments for every microbatch."""
        M, b, T1 = tokens.shape
        if M != self.M or b != self.b or T1 != self.T + 1:
            raise ValidationError(f"tokens shape {tuple(tokens.shape)} != ({self.M}, {self.b}, {self.T + 1})")
        ids = tokens[:, :, :-1].reshape(M, -1).to(torch.int32)
        tgt = tokens[:, :, 1:].reshape(M, -1).to(torch.int32)
        segs = [native.embed_segments(ids[mb]) for mb in range(M)]
        pin = lambda t: t.contiguous().pin_memory()  # noqa: E731
        return {"ids": pin(ids), "tgt": pin(tgt), "perm": pin(torch.stack([s_[0] for s_ in segs])),
                "seg_start": pin(torch.stack([s_[1] for s_ in segs])), "seg_id": pin(torch.stack([s_[2] for s_ in segs])),
                "n_seg": pin(torch.stack([s_[3] for s_ in segs]))}

    def h2d_bytes(self, tokens: torch.Tensor) -> int:
        M = tokens.shape[0]
        n = self.n
        return M * 4 * (n + n + n + (n + 1) + n + 1)

    def step(self, tokens: torch.Tensor, *, timing: bool = False) -> dict:
        """One synchronous training iteration over M microbatches.  Returns loss (host float)."""
        host = tokens if isinstance(tokens, dict) else self._stage_inputs(tokens)
        self.step_count += 1
        dev0 = self.devices[0]
        ev = {}
        t_iter0 = torch.cuda.Event(enable_timing=True)
        t_iter1 = torch.cuda.Event(enable_timing=True)
        for d in self.devices:
            self.streams[d].wait_stream(torch.cuda.current_stream(d))
        t_iter0.record(self.streams[dev0])
        for (st, d), ps in self.psets.items():
            with torch.cuda.stream(self.streams[d]):
                ps.g.zero_()
        executed = []
        for op in self.ops:
            v, slot, mb = op.node, op.slot, op.mb
            dev = self.placement[v]
            s = self.streams[dev]
            sb = self.slots[(v, slot)]
            if op.kind == F and op.pos == 0:
                _h2d(sb.ids, host["ids"][mb], s)
            if op.kind == L:
                _h2d(sb.targets, host["tgt"][mb], s)
            if op.kind == B and op.pos == 0:
                _h2d(sb.perm, host["perm"][mb], s)
                _h2d(sb.seg_start, host["seg_start"][mb], s)
                _h2d(sb.seg_id, host["seg_id"][mb], s)
                _h2d(sb.n_seg, host["n_seg"][mb], s)
            if timing:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
            if self.use_graphs:
                with torch.cuda.device(dev), torch.cuda.stream(s):
                    self._graphs[(op.kind, v, slot)].replay()   # replays on the current stream
                out = self._bwd_out[(op.kind, v, slot)]
            else:
                with torch.cuda.device(dev):
                    out = self._run_op(op.kind, v, slot, s)
            if timing:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(s)
                ev[len(executed)] = (e0, e1)
            executed.append((op.kind, v, op.agent, op.wave))
            self._hop(op, out, s)
            if op.kind == L:
                with torch.cuda.stream(s):
                    self.mb_loss[mb:mb + 1].copy_(sb.loss, non_blocking=True)
        self.optimizer_step()
        t_iter1.record(self.streams[dev0])
        for d in self.devices:
            torch.cuda.current_stream(d).wait_stream(self.streams[d])
        loss = float(self.mb_loss.sum().item()) / self.M
        out = {"loss": loss, "executed": executed}
        if timing:
            torch.cuda.synchronize()
            out["iter_ms"] = t_iter0.elapsed_time(t_iter1)
            out["op_times"] = {i: (t_iter0.elapsed_time(a), t_iter0.elapsed_time(b_)) for i, (a, b_) in ev.items()}
        return out

    def _hop(self, op, out, s):
        """Send the op's output to the next node on the microbatch's path (spx_hop)."""
        nodes = self.paths[op.agent]
        last = len(nodes) - 1
        src_dev = self.placement[op.node]
        if op.kind == F:
            if op.pos < last:
                nv = nodes[op.pos + 1]
                dst = self.slots[(nv, self._slot_of[(op.mb, nv)])].xs[0]
            else:
                nv = nodes[0]
                dst = self.slots[(nv, self._slot_of[(op.mb, nv)])].ret
        elif op.kind == L:
            nv = nodes[last]
            dst = self.slots[(nv, self._slot_of[(op.mb, nv)])].gin
        else:
            if op.pos == 0:
                return
            nv = nodes[op.pos - 1]
            dst = self.slots[(nv, self._slot_of[(op.mb, nv)])].gin
        dst_dev = self.placement[nv]
        native.hop(dst, dst_dev, out, src_dev, out.numel() * out.element_size(), stream=s)
        if dst_dev != src_dev:
            e = torch.cuda.Event()
            e.record(s)
            self.streams[dst_dev].wait_event(e)

    def launches_per_step(self) -> int:
        """libspx kernel launches in one iteration (graph contents + optimizer); needs graphs."""
        if not self.use_graphs:
            raise ValidationError("launch accounting needs use_graphs=True")
        if not self._opt_launches:
            n0 = native.launches()
            self._opt_launch_probe()
            self._opt_launches = native.launches() - n0
        return sum(self._graph_launches[(op.kind, op.node, op.slot)] for op in self.ops) + self._opt_launches

    def gemm_counts_per_step(self) -> dict:
        """GEMM key -> launches per iteration (recorded at capture when native.record_gemms(True))."""
        out: dict = {}
        for op in self.ops:
            for key in self._graph_gemms.get((op.kind, op.node, op.slot), []):
                out[key] = out.get(key, 0) + 1
        return out

    def _opt_launch_probe(self):
        # 2 (sumsq) per distinct stage + 1 (clip) + 1 (adamw) per parameter set
        native._count(2 * len({st for st, _ in self.psets}) + 1 + len(self.psets))

    def optimizer_step(self):
        """Replica sync (only across devices), global-norm clip, AdamW — all on device."""
        o = self.optim
        dev0 = self.devices[0]
        self.sync_grads()
        s0 = self.streams[dev0]
        for d in self.devices:
            if d != dev0:
                e = torch.cuda.Event()
                e.record(self.streams[d])
                s0.wait_event(e)
        # each stage counted once in the global norm
        seen = set()
        idx = 0
        for (st, d), ps in sorted(self.psets.items()):
            if st in seen:
                continue
            seen.add(st)
            with torch.cuda.device(d):
                native.sumsq(ps.g, ps.lay.numel, self._sumsq_ws[d], self._sumsq[dev0][idx:idx + 1] if d == dev0
                             else self._sumsq[d][idx:idx + 1], stream=self.streams[d])
            idx += 1
        with torch.cuda.device(dev0):
            native.clip_scale(self._sumsq[dev0], idx, o.max_grad_norm, self._clip[dev0], self._norm[dev0], stream=s0)
        for (st, d), ps in sorted(self.psets.items()):
            with torch.cuda.device(d):
                native.adamw(ps.p32, ps.g, ps.m, ps.v, ps.pbf, n=ps.lay.numel, n_decay=ps.lay.n_decay, lr=o.lr,
                             beta1=o.beta1, beta2=o.beta2, eps=o.eps, weight_decay=o.weight_decay,
                             step=self.step_count, grad_scale=self._clip[d], stream=self.streams[d])

    def sync_grads(self):
        """Sum gradients of replica parameter sets that live on different devices (single-process
        multi-GPU path; the multi-process path uses NCCL all-reduce, see dist_trainer)."""
        by_stage: dict[int, list] = {}
        for (st, d), ps in sorted(self.psets.items()):
            by_stage.setdefault(st, []).append(ps)
        for st, sets in by_stage.items():
            if len(sets) < 2:
                continue
            raise NotImplementedError("single-process multi-GPU replicas: use dist_trainer (one process per GPU)")

    # ---- inspection (tests) ----
    def grads(self) -> list[dict[str, torch.Tensor]]:
        """Per-stage canonical fp32 gradients of the last iteration (pre-clip), summed over
        co-resident replicas."""
        torch.cuda.synchronize()
        out = []
        for st in range(self.assignment.s):
            sets = [ps for (s_, d), ps in self.psets.items() if s_ == st]
            g = sum(ps.g.double().cpu() for ps in sets).float()
            out.append(unpack_stage(self.cfg, self.layouts[st], g))
        return out

    def params(self) -> list[dict[str, torch.Tensor]]:
        torch.cuda.synchronize()
        out = []
        for st in range(self.assignment.s):
            ps = next(ps for (s_, d), ps in sorted(self.psets.items()) if s_ == st)
            out.append(unpack_stage(self.cfg, self.layouts[st], ps.p32))
        return out

    def grad_norm(self) -> float:
        torch.cuda.synchronize()
        return float(self._norm[self.devices[0]].item())


def _h2d(dst: torch.Tensor, src: torch.Tensor, stream) -> None:
    with torch.cuda.stream(stream):
        dst.copy_(src, non_blocking=True)


def execute(schedule: Schedule, topology: Topology, sim_config: SimConfig, model_cfg: ModelConfig, placement,
            tokens: torch.Tensor, *, assignment, b: int, split=None, seed: int = 0, steps: int = 1,
            use_graphs: bool = True) -> ExecReport:
    """Run ``steps`` iterations of the schedule on the GPU(s); report the last one measured."""
    tr = Trainer(schedule, topology, sim_config, model_cfg, assignment, b=b, T=tokens.shape[-1] - 1, split=split,
                 placement=placement, seed=seed, use_graphs=use_graphs)
    res = None
    for _ in range(steps):
        res = tr.step(tokens, timing=True)
    return tr.make_report(res)


def _make_report(self: Trainer, res: dict) -> ExecReport:
    n = self.topology.n
    busy = [0.0] * n
    order: dict[int, list] = {}
    trace = []
    start_f0: dict[int, float] = {}
    e2e = [0.0] * self.M
    wait = 0.0
    ready_at: dict = {}
    for i, (kind, v, agent, wave) in enumerate(res["executed"]):
        t0, t1 = res["op_times"][i]
        busy[v] += t1 - t0
        order.setdefault(v, []).append((kind, agent, wave))
        trace.append((t0, v, "start", agent, wave, {"F": "fwd", "L": "loss", "B": "bwd"}[kind]))
        trace.append((t1, v, "end", agent, wave, {"F": "fwd", "L": "loss", "B": "bwd"}[kind]))
        op = self.ops[i]
        if kind == F and op.pos == 0:
            start_f0[op.mb] = t0
        if kind == B and op.pos == 0:
            e2e[op.mb] = t1 - start_f0[op.mb]
    mk = res["iter_ms"]
    return ExecReport(iteration_makespan=mk, microbatch_e2e=e2e, total_collision_wait=wait, node_busy=busy,
                      node_idle=[mk - x for x in busy], loss=res["loss"], mb_loss=self.mb_loss.tolist(),
                      grad_norm=self.grad_norm(), node_order=order, trace=trace)


Trainer.make_report = _make_report
