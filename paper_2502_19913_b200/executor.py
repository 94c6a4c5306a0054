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

LW = "LW"  # graph key kind: the head weight gradient that follows an L op (off the backward chain)
from .topology import Topology

BF16 = torch.bfloat16
F32 = torch.float32
# the attention backward's D = rowsum(dO*O) pass fused into the O-projection dgrad (head_dim 64/128);
# SPX_ATTN_DELTA_FUSED=0 keeps the separate pass (benchmarking)
_DELTA_FUSED = os.environ.get("SPX_ATTN_DELTA_FUSED", "1") != "0"


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
                                         # (ops whose producer ran on this rank; see make_report)
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


class NodeParams:
    """A logical node's handle on its stage's parameter set with a private gradient buffer.

    With one compute stream per logical node, co-resident replicas of a stage run concurrently, so
    they accumulate into separate buffers; the optimizer adds them in node order (deterministic).
    The first hosted node of a stage uses the parameter set's own gradient buffer."""

    def __init__(self, ps: ParamSet, g: torch.Tensor):
        self.ps, self.g, self.lay = ps, g, ps.lay

    def w(self, name):
        return self.ps.w(name)

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
        # gradient w.r.t. this node's input (the B op's output, sent to the previous node); slot-
        # owned so a cross-GPU send can drain asynchronously on the send stream
        self.gout = torch.empty(n, cfg.d, **e) if not origin else None
        if origin:
            self.tok = torch.zeros(b, T + 1, dtype=torch.int64, device=device)  # raw token block
            self.ids = torch.zeros(n, dtype=torch.int32, device=device)
            self.targets = torch.zeros(n, dtype=torch.int32, device=device)
            self.perm = torch.zeros(n, dtype=torch.int32, device=device)
            self.seg_start = torch.zeros(n + 1, dtype=torch.int32, device=device)
            self.seg_id = torch.zeros(n, dtype=torch.int32, device=device)
            self.n_seg = torch.zeros(1, dtype=torch.int32, device=device)
            self.ret = torch.empty(n, cfg.d, **e)       # activation returned to the origin (L input)
            self.dret = torch.empty(n, cfg.d, **e)      # L output: gradient sent to the last node
            self.loss = torch.zeros(1, dtype=F32, device=device)


class Scratch:
    """Per-device scratch shared by all ops of that device (ops are serialised on its stream)."""

    def __init__(self, cfg: ModelConfig, n: int, b: int, T: int, device, with_head: bool):
        d, f = cfg.d, cfg.ffn
        e = dict(dtype=BF16, device=device)
        # Buffers read by a layer's weight-gradient group are double-buffered by layer parity (the
        # group of layer i may still run while layer i-1 computes), and the layer-output gradients
        # rotate through three buffers (layer i's dy is read by its group until layer i-2 starts).
        self.dx = [torch.empty(n, d, **e) for _ in range(3)]
        self.dxm2 = [torch.empty(n, d, **e) for _ in range(2)]
        self.dxn = torch.empty(n, d, **e)
        self.dh = torch.empty(n, f, **e)
        self.dgu2 = [torch.empty(n, 2 * f, **e) for _ in range(2)]
        self.do = torch.empty(n, cfg.n_heads * cfg.head_dim, **e)
        self.dqkv2 = [torch.empty(n, cfg.qkv_dim, **e) for _ in range(2)]
        self.delta = torch.empty(native.attn_bwd_ws_floats(b, cfg.n_heads, T, cfg.head_dim, cfg.n_kv_heads), dtype=F32,
                                 device=device)
        self.rms_ws = torch.empty(native.rmsnorm_ws_floats(n, d), dtype=F32, device=device)
        self.rope = rope_cos_sin(T, cfg.head_dim, cfg.rope_theta).to(device)
        if with_head:
            self.xf = torch.empty(n, d, **e)
            self.rstdf = torch.empty(n, dtype=F32, device=device)
            self.logits = torch.empty(n, cfg.vocab, **e)
            # cross-entropy partials of the head GEMM epilogue: per row, (max, sum exp) of each
            # 128-column block of the logits (EPI_XENT; V % 128 == 0)
            self.xent_nb = cfg.vocab // 128 if cfg.vocab % 128 == 0 else 0
            self.xparts = torch.empty(n, 2 * max(1, self.xent_nb), dtype=F32, device=device)
            self.row_loss = torch.empty(n, dtype=F32, device=device)
            self.dxf = torch.empty(n, d, **e)


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
        if hd in (64, 128):
            native.gemm_rope(a.xn1, ps.w(f"l{i}.wqkv"), a.qkv, M=n, N=qd, K=d, lda=d, ldb=d, ldc=qd, cos_sin=sc.rope,
                             rope_cols=(c.n_heads + c.n_kv_heads) * hd, T=self.T, head_dim=hd, stream=s)
        else:
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

    def layer_bwd(self, ps: ParamSet, i: int, x, a: LayerActs, dy, dx, sc: Scratch, s, side=None):
        """dy: grad of the layer output; dx: grad of the layer input (may not alias dy).

        The data-gradient chain runs on ``s``.  The four weight-gradient GEMMs (few output tiles,
        long K = tokens) form ONE grouped launch (spx_gemm_f32_group) issued as soon as their last
        input (dqkv) exists: on ``side`` when given -- forked from ``s`` and returned as an event
        the caller joins one layer later, so the group overlaps the next layer's data-gradient
        chain -- else inline on ``s``.  The buffers it reads are per-parity scratch (Scratch)."""
        c, n = self.cfg, self.n
        d, f, qd, hd = c.d, c.ffn, c.qkv_dim, c.head_dim
        od = c.n_heads * hd
        par = i & 1
        dgu, dxm, dqkv = sc.dgu2[par], sc.dxm2[par], sc.dqkv2[par]
        # MLP
        native.gemm(dy, ps.w(f"l{i}.wdown"), sc.dh, M=n, N=f, K=d, lda=d, ldb=f, ldc=f, b_mn=True, stream=s)
        native.swiglu_bwd(a.gu, sc.dh, dgu, rows=n, F=f, stream=s)
        native.gemm(dgu, ps.w(f"l{i}.wgu"), sc.dxn, M=n, N=d, K=2 * f, lda=2 * f, ldb=d, ldc=d, b_mn=True, stream=s)
        native.rmsnorm_bwd(a.xmid, ps.w(f"l{i}.mlp_norm"), a.rstd2, sc.dxn, dy, dxm, ps.gv(f"l{i}.mlp_norm"),
                           sc.rms_ws, rows=n, d=d, stream=s)
        # attention; dq, dk leave the attention backward already un-rotated (inverse RoPE fused)
        fused_delta = hd in (64, 128) and _DELTA_FUSED
        if fused_delta:  # D = rowsum(dO*O) in the O-projection dgrad's epilogue
            native.gemm_attn_delta(dxm, ps.w(f"l{i}.wo"), sc.do, a.o, a.lse, sc.delta, M=n, N=od, K=d, lda=d, ldb=od,
                                   ldc=od, ld_o=od, batch=self.b, T=self.T, head_dim=hd, stream=s)
        else:
            native.gemm(dxm, ps.w(f"l{i}.wo"), sc.do, M=n, N=od, K=d, lda=d, ldb=od, ldc=od, b_mn=True, stream=s)
        native.attn_bwd(a.qkv, a.o, sc.do, a.lse, sc.delta, dqkv, B=self.b, T=self.T, H=c.n_heads,
                        Hkv=c.n_kv_heads, hd=hd, ld_qkv=qd, ld_o=od, scale=self.scale, rope_cs=sc.rope,
                        delta_ready=fused_delta, stream=s)
        # weight gradients dW = dY^T X (both operands MN-major), accumulated in fp32
        group = [
            dict(A=dgu, B=a.xn2, C=ps.gv(f"l{i}.wgu"), M=2 * f, N=d, K=n, lda=2 * f, ldb=d, ldc=d, beta=1.0),
            dict(A=dqkv, B=a.xn1, C=ps.gv(f"l{i}.wqkv"), M=qd, N=d, K=n, lda=qd, ldb=d, ldc=d, beta=1.0),
            dict(A=dy, B=a.h, C=ps.gv(f"l{i}.wdown"), M=d, N=f, K=n, lda=d, ldb=f, ldc=f, beta=1.0),
            dict(A=dxm, B=a.o, C=ps.gv(f"l{i}.wo"), M=d, N=od, K=n, lda=d, ldb=od, ldc=od, beta=1.0),
        ]
        done = None
        if side is None:
            native.gemm_f32_group(group, stream=s)
        else:
            ev = torch.cuda.Event()
            ev.record(s)
            side.wait_event(ev)
            native.gemm_f32_group(group, stream=side)
            done = torch.cuda.Event()
            done.record(side)
        native.gemm(dqkv, ps.w(f"l{i}.wqkv"), sc.dxn, M=n, N=d, K=qd, lda=qd, ldb=d, ldc=d, b_mn=True, stream=s)
        native.rmsnorm_bwd(x, ps.w(f"l{i}.attn_norm"), a.rstd1, sc.dxn, dxm, dx, ps.gv(f"l{i}.attn_norm"),
                           sc.rms_ws, rows=n, d=d, stream=s)
        return done

    # ---- node ops ----
    def fwd(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, origin: bool, s, n_layers: int | None = None):
        """Embedding (at the origin) and the stage's layers; ``n_layers`` runs only the first ones
        (a partial stage, inference only).  Returns the output buffer."""
        if origin:
            native.embed_fwd(sb.ids, ps.w("embed"), sb.xs[0], n=self.n, d=self.cfg.d, stream=s)
        k = len(sb.layers) if n_layers is None else n_layers
        for i in range(k):
            self.layer_fwd(ps, i, sb.xs[i], sb.layers[i], sb.xs[i + 1], sc, s)
        return sb.xs[k]

    def head_xent(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, s, scale: float):
        """Head GEMM + cross-entropy: the GEMM epilogue (EPI_XENT) writes the
        bf16 logits and per-128-column (max, sum exp) partials; one pass then forms each row's
        log-sum-exp and loss and, for training (scale != 0), overwrites the logits with
        dlogits = (softmax - onehot) * scale.  Vocabularies that are not a multiple of 128 take
        the separate xent pass."""
        c, n, V = self.cfg, self.n, self.cfg.vocab
        if sc.xent_nb:
            native.gemm(sc.xf, ps.w("head"), sc.logits, M=n, N=V, K=c.d, lda=c.d, ldb=c.d, ldc=V,
                        epilogue=native.EPI_XENT, C2=sc.xparts, ldc2=2 * sc.xent_nb, stream=s)
            native.xent_from_parts(sc.logits, sc.xparts, sb.targets, sc.row_loss, nb=sc.xent_nb, n=n, V=V, ld=V,
                                   scale=scale, stream=s)
        else:
            native.gemm(sc.xf, ps.w("head"), sc.logits, M=n, N=V, K=c.d, lda=c.d, ldb=c.d, ldc=V, stream=s)
            native.xent_fwd_bwd(sc.logits, sb.targets, sc.row_loss, n=n, V=V, ld=V, scale=scale, stream=s)
        native.sum_f32(sc.row_loss, n, sb.loss, scale=1.0 / n, stream=s)

    def loss_fwd(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, s):
        """Inference loss at the origin: final norm, head, token-mean cross-entropy into sb.loss
        (no dlogits, no gradient is touched)."""
        c, n = self.cfg, self.n
        native.rmsnorm_fwd(sb.ret, ps.w("final_norm"), sc.xf, sc.rstdf, rows=n, d=c.d, eps=c.eps, stream=s)
        self.head_xent(ps, sb, sc, s, 0.0)

    def bwd(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, origin: bool, s, side=None):
        """Returns the buffer holding the gradient w.r.t. the node's input."""
        dy = sb.gin
        k = 0
        pending = {}  # layer -> its weight-gradient group's completion event (side stream)
        for i in reversed(range(len(sb.layers))):
            if i + 2 in pending:  # layer i reuses the parity-(i & 1) scratch and dx buffer of layer i+2
                s.wait_event(pending.pop(i + 2))
            dx = sb.gout if (i == 0 and sb.gout is not None) else sc.dx[k]
            done = self.layer_bwd(ps, i, sb.xs[i], sb.layers[i], dy, dx, sc, s, side)
            if done is not None:
                pending[i] = done
            dy, k = dx, (k + 1) % 3
        for ev in pending.values():  # join: all weight gradients of the node accumulated
            s.wait_event(ev)
        if origin:
            native.embed_bwd(sb.perm, sb.seg_start, sb.seg_id, sb.n_seg, self.n, dy, ps.gv("embed"), d=self.cfg.d,
                             stream=s)
        return dy

    def loss(self, ps: ParamSet, sb: SlotBuffers, sc: Scratch, s):
        """Final norm, de-embedding, cross-entropy fwd+bwd at the origin."""
        c, n = self.cfg, self.n
        d, V = c.d, c.vocab
        native.rmsnorm_fwd(sb.ret, ps.w("final_norm"), sc.xf, sc.rstdf, rows=n, d=d, eps=c.eps, stream=s)
        self.head_xent(ps, sb, sc, s, 1.0 / (n * self.M))
        native.gemm(sc.logits, ps.w("head"), sc.dxf, M=n, N=d, K=V, lda=V, ldb=d, ldc=d, b_mn=True, stream=s)
        native.rmsnorm_bwd(sb.ret, ps.w("final_norm"), sc.rstdf, sc.dxf, None, sb.dret, ps.gv("final_norm"),
                           sc.rms_ws, rows=n, d=d, stream=s)
        return sb.dret

    def loss_wgrad(self, ps: ParamSet, sc: Scratch, s):
        """The head's weight gradient from the L op's dlogits / normalised input.  Issued after the
        L op's hop, so the returned gradient leaves for the path's last node without waiting for
        this GEMM (it is off the backward chain; sc.logits / sc.xf are only rewritten by the node's
        next L op, later on the same stream)."""
        c, n = self.cfg, self.n
        native.gemm(sc.logits, sc.xf, ps.gv("head"), M=c.vocab, N=c.d, K=n, lda=c.vocab, ldb=c.d, ldc=c.d,
                    a_mn=True, b_mn=True, epilogue=native.EPI_F32, beta=1.0, stream=s)


# ---------------------------------------------------------------------------------------
# the trainer
# ---------------------------------------------------------------------------------------
def default_placement(n_nodes: int, n_ranks: int) -> list[int]:
    """Logical node i -> rank i mod n_ranks.  With contiguous stage numbering (stage st = nodes
    [st·r, (st+1)·r)) this puts the replicas of a stage on different ranks and gives every rank
    the same mix of S₀ and non-S₀ nodes (S₀ is the heavy stage)."""
    return [i % n_ranks for i in range(n_nodes)]


def balanced_placement(report: SimReport, n_nodes: int, n_ranks: int) -> list[int]:
    """Longest-processing-time placement of logical nodes onto ranks by the simulator's per-node
    busy time (F + L + B over the whole iteration).  The scheduler is placement-blind on a uniform
    NVSwitch box, so its paths can load replica nodes unevenly; co-resident nodes of one stage then
    share a parameter set.  Deterministic: ties go to the lower node / rank id."""
    busy = list(report.node_busy) + [0.0] * (n_nodes - len(report.node_busy))
    load = [0.0] * n_ranks
    out = [0] * n_nodes
    for v in sorted(range(n_nodes), key=lambda v: (-round(busy[v], 9), v)):
        r = min(range(n_ranks), key=lambda r: (round(load[r], 9), r))
        out[v] = r
        load[r] += busy[v]
    return out


def allreduce_points(ops, node_stage: list[int], stages) -> dict:
    """Global op index -> replicated stages whose all-reduce is issued right after that op: the
    stage's last op in the global order.  A function of the op list only, so every rank issues
    its replica all-reduces (and, interleaved, its NCCL hops) in one consistent order -- NCCL
    kernels of different communicators enqueued in different orders on two ranks can deadlock."""
    out: dict = {}
    for st in sorted(stages):
        last = max(i for i, op in enumerate(ops) if node_stage[op.node] == st)
        out.setdefault(last, []).append(st)
    return out


def static_slots(schedule: Schedule, n_nodes: int) -> tuple[dict, list[int]]:
    """Activation slot of every (agent, node): the agent's rank among the agents whose path visits
    the node.  A slot is then only ever reused by the *same* agent's next wave, which launches
    after the previous wave's backward has left every node of the path, so a
    path hop may write its destination slot as soon as the producer op is done, without racing
    the previous owner.  Under TC1 (≤ m paths per node) this needs ≤ m slots per node."""
    users: dict[int, list[int]] = {v: [] for v in range(n_nodes)}
    for a in sorted(schedule.paths):
        for v in schedule.paths[a].nodes:
            users[v].append(a)
    slot_of = {(a, v): users[v].index(a) for v in users for a in users[v]}
    return slot_of, [max(1, len(users[v])) for v in range(n_nodes)]


def hop_plan(ops, paths: dict, placement: list[int]) -> list:
    """Per op (global order): the path hop that follows it, or None at the end of a path.

    Entry = (dst_node, buffer, src_rank, dst_rank, consumer_kind): F feeds the next node's F (its
    layer-0 input ``xs0``) or, after the last stage, the origin's loss op (``ret``); L feeds the
    last node's B (``gin``); B feeds the previous node's B.  Every rank derives the same plan from
    the same simulator ops, so sends and receives between any two ranks are posted in the same
    (global) order on both sides."""
    out = []
    for op in ops:
        nodes = paths[op.agent]
        last = len(nodes) - 1
        if op.kind == F:
            dst = (nodes[op.pos + 1], "xs0", F) if op.pos < last else (nodes[0], "ret", L)
        elif op.kind == L:
            dst = (nodes[last], "gin", B)
        else:
            dst = (nodes[op.pos - 1], "gin", B) if op.pos > 0 else None
        out.append(None if dst is None else (dst[0], dst[1], placement[op.node], placement[dst[0]], dst[2]))
    return out


class Trainer:
    """Weights, optimizer state, activation slots and captured graphs for one config on one rank.

    ``rank``/``world``: one process per GPU (torch.distributed, NCCL).  ``placement[v]`` is the
    rank that hosts logical node v.  Every rank builds the same schedule and simulator op list and
    walks it in the same global order: it runs the ops of its own nodes, sends a path hop to the
    rank of the next node and posts the matching receive for hops that target its nodes; a local
    ``spx_hop`` copy when both nodes are on this rank.  ``hop_transport`` (default "peer", env
    SPX_HOP): "peer" pushes the activation straight into the consumer's slot over NVLink peer
    memory (spx_hop_push / spx_hop_wait on CUDA-IPC-mapped buffers and arrival flags); "nccl"
    uses NCCL send/recv on a per-rank-pair communicator.  With world=1 (the default) everything is
    on cuda:<device> and every hop is a local copy."""

    def __init__(self, schedule: Schedule, topology: Topology, sim_config: SimConfig, cfg: ModelConfig,
                 assignment, *, b: int, T: int | None = None, split: list[int] | None = None,
                 placement: list[int] | None = None, seed: int = 0, optim: OptimConfig | None = None,
                 use_graphs: bool = True, params: list | None = None, rank: int = 0, world: int = 1,
                 device: int | None = None, hop_transport: str | None = None, keep_grads: bool = False):
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
        # keep_grads=False (default): AdamW clears each gradient it consumed and co-resident
        # replica buffers are cleared by their merge, so no fill pass runs per iteration.
        # keep_grads=True keeps the last iteration's gradients readable (grads(); tests) and zeroes
        # them at the start of the next step instead; the updates are bit-identical.
        self.keep_grads = keep_grads
        self.node_stage = assignment.node_stage()
        self.rank, self.world = rank, world
        self.hop_transport = hop_transport or os.environ.get("SPX_HOP", "peer")
        if self.hop_transport not in ("peer", "nccl"):
            raise ValidationError(f"hop_transport must be 'peer' or 'nccl', not {self.hop_transport!r}")
        # peer hops as an SM push kernel ("sm": SPX_HOP_CTAS CTAs, each +1 on the flag; 8 MiB in
        # 21 us) or on the copy engine ("ce": no SMs, then a one-thread flag kernel; 27 us, the
        # gap before the flag kernel costs more than the faster copy saves).  Same step time.
        self.hop_engine = os.environ.get("SPX_HOP_ENGINE", "sm")
        if self.hop_engine not in ("ce", "sm"):
            raise ValidationError(f"SPX_HOP_ENGINE must be 'ce' or 'sm', not {self.hop_engine!r}")
        self.hop_ctas = int(os.environ.get("SPX_HOP_CTAS", "32"))
        self.hop_timeout_s = float(os.environ.get("SPX_HOP_TIMEOUT_S", "120"))
        self.hop_inc = 1 if self.hop_engine == "ce" else self.hop_ctas
        self.report: SimReport = simulate(schedule, topology, sim_config)
        if placement is None:
            placement = balanced_placement(self.report, topology.n, world)
        self.placement = list(placement)
        if len(self.placement) != topology.n or max(self.placement) >= world:
            raise ValidationError(f"placement {self.placement} does not map {topology.n} nodes onto {world} ranks")
        self.dev = torch.device("cuda", rank if device is None else device)
        # Op order.  The simulator gives every logical node its own device; with several nodes per
        # GPU each rank replays its nodes' ops on one stream, so the order matters.  The order of a
        # simulation that shares each GPU among its nodes (SimConfig.device_of) is used when it
        # replays faster (simulator.replay_makespan): C3 / C4 at 4 GPUs 6-12 % shorter by this
        # estimate, C2 about the same.  Every rank computes the same choice.
        self.order_kind = "simulated"
        if world > 1 and len(set(self.placement)) < topology.n and os.environ.get("SPX_COLOC_ORDER", "1") != "0":
            from dataclasses import replace as _replace

            from .simulator import replay_makespan

            co = simulate(schedule, topology, _replace(sim_config, device_of=tuple(self.placement)))
            t_pure = replay_makespan(self.report.ops, schedule, topology, sim_config, self.placement)
            t_co = replay_makespan(co.ops, schedule, topology, sim_config, self.placement)
            if t_co < t_pure:
                self.report, self.order_kind = co, "colocated"
        self.ops = self.report.ops
        self.step_count = 0
        self.use_graphs = use_graphs
        self.agents = sorted(a.id for a in schedule.agents)
        self.paths = {a: schedule.paths[a].nodes for a in self.agents}
        self.slot_of, self.n_slots = static_slots(schedule, topology.n)
        self.hops = hop_plan(self.ops, self.paths, self.placement)
        origin: dict = {}
        for op in self.ops:  # token_prep at F pos 0 feeds the L and B pos 0 ops of the same origin slot
            if (op.kind == F and op.pos == 0) or op.kind == L or (op.kind == B and op.pos == 0):
                if origin.setdefault((op.agent, op.wave), op.node) != op.node:
                    raise ValidationError(f"agent {op.agent} wave {op.wave}: embed, loss and embed-backward "
                                          f"ops on different nodes")
        self.my_nodes = [v for v in range(topology.n) if self.placement[v] == rank]
        self.my_stages = sorted({self.node_stage[v] for v in self.my_nodes})
        self.stage_ranks = {st: sorted({self.placement[v] for v in range(topology.n) if self.node_stage[v] == st})
                            for st in range(assignment.s)}

        with torch.cuda.device(self.dev):
            if params is not None:
                got = [sum(1 for k in p if k.endswith(".wq")) for p in params]
                if got != list(self.split):
                    raise ValidationError(f"params hold {got} layers per stage, the layer split is {self.split} "
                                          f"(pass split=)")
            canon = params if params is not None else init_params(cfg, self.split, seed)
            self.layouts = [stage_layout(cfg, st, self.split) for st in range(assignment.s)]
            # one parameter set per stage hosted here (co-resident replicas share it)
            self.psets = {st: ParamSet(cfg, self.layouts[st], pack_stage(cfg, self.layouts[st], canon[st]), self.dev)
                          for st in self.my_stages}
            self.slots: dict[tuple[int, int], SlotBuffers] = {}
            for v in self.my_nodes:
                for j in range(self.n_slots[v]):
                    self.slots[(v, j)] = SlotBuffers(cfg, self.split[self.node_stage[v]], self.node_stage[v] == 0,
                                                     self.n, b, self.T, self.dev)
            # One compute stream (+ weight-gradient side stream), scratch set and gradient buffer per
            # hosted logical node: a node's ops wait only for their own inputs and concurrent nodes
            # fill each other's kernel tails.  Default on a single GPU (the iteration is throughput
            # bound: 289 vs 310 ms at C2).  Across GPUs the simulator's global order on one stream
            # is faster (concurrency slows the pipeline's critical ops: 4 GPUs 124 vs 116 ms), so
            # there every op of a rank is serialised on one stream.  SPX_NODE_STREAMS=0/1 forces.
            env = os.environ.get("SPX_NODE_STREAMS")
            self.node_streams = (world == 1) if env is None else env != "0"
            side_on = os.environ.get("SPX_WGRAD_SIDE", "1") != "0"
            # one shared scratch set when every op of the rank is serialised on one stream
            self.scratch = None if self.node_streams else \
                Scratch(cfg, self.n, b, self.T, self.dev, with_head=0 in self.my_stages)
            self.nparams: dict[int, NodeParams] = {}
            self.extra_grads: dict[int, list] = {st: [] for st in self.my_stages}
            for v in self.my_nodes:
                st = self.node_stage[v]
                ps = self.psets[st]
                if not self.node_streams or not any(self.nparams[u].ps is ps for u in self.nparams):
                    self.nparams[v] = NodeParams(ps, ps.g)
                else:
                    g = torch.zeros_like(ps.g)
                    self.extra_grads[st].append(g)
                    self.nparams[v] = NodeParams(ps, g)
            # No split-K workspace: the weight-gradient GEMMs run on a side stream next to the
            # data-gradient chain, which uses the SMs a wgrad leaves idle; split-K's partial
            # traffic costs more SM time than it saves there (spx_gemm_set_workspace, spx.h).
            native.gemm_set_workspace(None)
            self.stream = torch.cuda.Stream(device=self.dev)
            self.recv_stream = torch.cuda.Stream(device=self.dev)
            self.send_stream = torch.cuda.Stream(device=self.dev)
            # weight-gradient GEMMs run on a side stream, forked/joined per layer inside the B graphs
            self.side_stream = torch.cuda.Stream(device=self.dev) if side_on else None
            # embedding-backward grouping (token sort) of each microbatch, off the compute streams
            self.prep_stream = torch.cuda.Stream(device=self.dev)
            self._prep_done: dict = {}
            if self.node_streams:
                self.nstream = {v: torch.cuda.Stream(device=self.dev) for v in self.my_nodes}
                self.nside = {v: (torch.cuda.Stream(device=self.dev) if side_on else None) for v in self.my_nodes}
                self.nscratch = {v: Scratch(cfg, self.n, b, self.T, self.dev, with_head=self.node_stage[v] == 0)
                                 for v in self.my_nodes}
                # hop streams per node too: a send / receive never queues behind another node's
                self.nsend = {v: torch.cuda.Stream(device=self.dev) for v in self.my_nodes}
                self.nrecv = {v: torch.cuda.Stream(device=self.dev) for v in self.my_nodes}
            else:
                self.nstream = {v: self.stream for v in self.my_nodes}
                self.nside = {v: self.side_stream for v in self.my_nodes}
                self.nscratch = {v: self.scratch for v in self.my_nodes}
                self.nsend = {v: self.send_stream for v in self.my_nodes}
                self.nrecv = {v: self.recv_stream for v in self.my_nodes}
            self.prog = StageProgram(cfg, self.n, b, self.T, self.M)
            self.mb_loss = torch.zeros(self.M, dtype=F32, device=self.dev)
            self._sumsq = torch.zeros(assignment.s, dtype=F32, device=self.dev)
            self._sumsq_ws = torch.empty(native.sumsq_ws_floats(), dtype=F32, device=self.dev)
            self._clip = torch.ones(1, dtype=F32, device=self.dev)
            self._norm = torch.zeros(1, dtype=F32, device=self.dev)
        self._graphs: dict = {}
        self._graph_launches: dict = {}
        self._graph_gemms: dict = {}
        self._opt_launches = 0
        self._outs: dict = {}
        self._groups: dict = {}
        self._ar_after: dict = {}
        if world > 1:
            self._init_comm()
        if use_graphs:
            self._capture_all()
        if world > 1:
            # no rank's first hop_wait may start while a slower rank is still capturing graphs
            import torch.distributed as dist

            dist.barrier()

    # ---- communication setup (multi-process) ----
    def _init_comm(self):
        import torch.distributed as dist

        # the hop protocol assumes every rank uses the same transport, engine and CTA count (the
        # receiver's expected flag count is hop_inc per hop): agree before anything branches on it
        mine = (self.hop_transport, self.hop_engine, self.hop_ctas, self.hop_timeout_s)
        allc = [None] * self.world
        dist.all_gather_object(allc, mine)
        if any(c != allc[0] for c in allc):
            raise ValidationError(f"hop settings differ across ranks (SPX_HOP, SPX_HOP_ENGINE, SPX_HOP_CTAS, "
                                  f"SPX_HOP_TIMEOUT_S): {allc}")
        native.hop_set_timeout(self.hop_timeout_s)
        # one libspx-owned NCCL communicator per replicated stage (spx_comm_init), created in stage
        # order on every rank (a global order, so the blocking inits cannot deadlock); the group's
        # lowest rank makes the unique id, every rank learns it from one all-gather
        uids = {st: native.comm_unique_id() for st in range(self.assignment.s)
                if len(self.stage_ranks[st]) > 1 and self.stage_ranks[st][0] == self.rank}
        alluid = [None] * self.world
        dist.all_gather_object(alluid, uids)
        for st in range(self.assignment.s):
            ranks = self.stage_ranks[st]
            if len(ranks) > 1 and self.rank in ranks:
                self._groups[st] = native.comm_init(alluid[ranks[0]][st], len(ranks), ranks.index(self.rank))
        # the replica all-reduce of a stage is issued, on its own stream, at the stage's last op in
        # the global op order -- the same walk position on every rank, so all NCCL work (these
        # all-reduces and NCCL hops) is enqueued in one consistent order across ranks (NCCL
        # kernels of different communicators issued in different orders can deadlock each
        # other); this rank's ops of the stage are all enqueued by then, and the all-reduce
        # overlaps the remaining ops
        self._ar_after = allreduce_points(self.ops, self.node_stage, self._groups)
        self._ar_stream = {st: torch.cuda.Stream(device=self.dev) for st in self._groups}
        # one process group (own NCCL communicator and stream) per rank pair for the path hops, so
        # hops between different pairs, and the replica all-reduces, never serialise behind each
        # other; created and warmed up in one global (lexicographic) order on every rank
        self._pair = {}
        for a in range(self.world):
            for b_ in range(a + 1, self.world):
                g = dist.new_group([a, b_])
                if self.rank in (a, b_):
                    self._pair[b_ if self.rank == a else a] = g
        buf = torch.zeros(1, device=self.dev)
        for a in range(self.world):
            for b_ in range(a + 1, self.world):
                if self.rank == a:
                    dist.send(buf, b_, group=self._pair[b_])
                    dist.recv(buf, b_, group=self._pair[b_])
                elif self.rank == b_:
                    dist.recv(buf, a, group=self._pair[a])
                    dist.send(buf, a, group=self._pair[a])
        torch.cuda.synchronize(self.dev)
        if self.hop_transport == "peer":
            self._init_peer_hops()

    def _init_peer_hops(self):
        """NVLink peer-memory hops: export this rank's hop-receive buffers (layer-0 input,
        returned activation, incoming gradient of every hosted slot) and one int32 arrival flag
        per buffer, map every peer's (spx_ipc_export / spx_ipc_open).  Dedupes allocations: a
        CUDA IPC handle may be opened once per process."""
        import torch.distributed as dist

        recv = []
        for (v, j), sb in sorted(self.slots.items()):
            recv.append(((v, j, "xs0"), sb.xs[0]))
            recv.append(((v, j, "gin"), sb.gin))
            if getattr(sb, "ret", None) is not None:
                recv.append(((v, j, "ret"), sb.ret))
        self._flags = torch.zeros(max(1, len(recv)), dtype=torch.int32, device=self.dev)
        self._flag_local = {k: self._flags.data_ptr() + 4 * i for i, (k, _) in enumerate(recv)}
        self._flag_expect = {k: 0 for k, _ in recv}
        # every step below is collective-safe: a rank whose CUDA IPC export or mapping fails
        # still takes part in the exchange, and then ALL ranks fall back to NCCL hops (loudly)
        err = None
        try:
            mine = {"flags": native.ipc_export(self._flags),
                    "bufs": {k: native.ipc_export(t) for k, t in recv}}
        except native.NativeError as e:
            mine, err = None, e
        allx = [None] * self.world
        dist.all_gather_object(allx, mine)
        self._ipc_bases: dict = {}
        self._peer_addr: dict = {}
        self._peer_flag: dict = {}

        def addr(hoff):
            h, off = hoff
            if h not in self._ipc_bases:
                self._ipc_bases[h] = native.ipc_open(h)
            return self._ipc_bases[h] + off

        if all(ex is not None for ex in allx):
            try:
                for r, ex in enumerate(allx):
                    if r == self.rank:
                        continue
                    fbase = addr(ex["flags"])
                    for i, (k, hoff) in enumerate(ex["bufs"].items()):
                        self._peer_addr[k] = addr(hoff)
                        self._peer_flag[k] = fbase + 4 * i
            except native.NativeError as e:
                err = e
        ok = torch.tensor([0 if err is not None or any(ex is None for ex in allx) else 1], device=self.dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if not int(ok.item()):
            import sys

            print(f"[spx] rank {self.rank}: NVLink peer hops unavailable ({err or 'a peer failed'}); "
                  "using NCCL send/recv hops", file=sys.stderr, flush=True)
            self._unmap_peers()
            self.hop_transport = "nccl"
        torch.cuda.synchronize(self.dev)
        dist.barrier()

    def _push(self, dst_addr: int, src, flag_addr: int, stream):
        """One cross-GPU hop into a peer-mapped slot, then its arrival-flag update."""
        nbytes = src.numel() * src.element_size()
        if self.hop_engine == "ce":
            native.hop_push_ce(dst_addr, src, nbytes, flag_addr, stream=stream)
        else:
            native.hop_push(dst_addr, src, nbytes, flag_addr, self.hop_ctas, stream=stream)

    def close(self):
        """Unmap peer allocations (peer hop transport) and free the replica communicators."""
        for comm in getattr(self, "_groups", {}).values():
            try:
                native.comm_destroy(comm)
            except Exception:
                pass
        self._groups = {}
        self._unmap_peers()

    def _unmap_peers(self):
        for base in getattr(self, "_ipc_bases", {}).values():
            try:
                native.ipc_close(base)
            except Exception:
                pass
        self._ipc_bases = {}

    def __del__(self):
        self.close()

    # ---- graph capture ----
    def _run_op(self, kind: str, v: int, slot: int, s):
        ps = self.nparams[v]
        sb = self.slots[(v, slot)]
        sc = self.nscratch[v]
        origin = self.node_stage[v] == 0
        if kind == F:
            self.prog.fwd(ps, sb, sc, origin, s)
            return sb.xs[-1]
        if kind == L:
            return self.prog.loss(ps, sb, sc, s)
        if kind == LW:
            self.prog.loss_wgrad(ps, sc, s)
            return None
        return self.prog.bwd(ps, sb, sc, origin, s, self.nside[v])

    def _key(self, op):
        return (op.kind, op.node, self.slot_of[(op.agent, op.node)])

    def _capture_all(self):
        keys = sorted({self._key(op) for op in self.ops if self.placement[op.node] == self.rank})
        keys += [(LW, v, slot) for (kind, v, slot) in keys if kind == L]
        with torch.cuda.device(self.dev):
            for key in keys:
                kind, v, slot = key
                g = torch.cuda.CUDAGraph()
                cs = self.nstream[v]
                cs.wait_stream(torch.cuda.current_stream())
                n0 = native.launches()
                native.take_gemm_log()
                with torch.cuda.graph(g, stream=cs):
                    out = self._run_op(kind, v, slot, torch.cuda.current_stream())
                self._graph_launches[key] = native.launches() - n0
                self._graph_gemms[key] = native.take_gemm_log()
                self._graphs[key] = g
                self._outs[key] = out
            torch.cuda.synchronize(self.dev)

    # ---- inputs ----
    def _stage_inputs(self, tokens: torch.Tensor):
        """The step's host input: the token blocks [M, b, T+1] (int64) in pinned memory.  Inputs,
        targets and the embedding-backward grouping are derived on the device (``token_prep``)."""
        M, b, T1 = tokens.shape
        if M != self.M or b != self.b or T1 != self.T + 1:
            raise ValidationError(f"tokens shape {tuple(tokens.shape)} != ({self.M}, {self.b}, {self.T + 1})")
        t = tokens.to(torch.int64).contiguous()
        if t.is_pinned():
            return {"tokens": t}
        # one persistent pinned staging buffer (pinning a fresh tensor every step costs more than
        # the copy); the previous step's H2D copies from it completed before that step returned
        # (its loss readback waits for every stream of the step)
        if getattr(self, "_pinned", None) is None:
            self._pinned = torch.empty_like(t).pin_memory()
        self._pinned.copy_(t)
        return {"tokens": self._pinned}

    def h2d_bytes(self, tokens: torch.Tensor) -> int:
        """Bytes of token blocks this rank copies host->device per iteration."""
        per = 8 * self.b * (self.T + 1)
        mine = sum(1 for op in self.ops if op.kind == F and op.pos == 0 and self.placement[op.node] == self.rank)
        return mine * per

    # ---- hop destinations ----
    def _dst_buffer(self, op, nv, name):
        sb = self.slots[(nv, self.slot_of[(op.agent, nv)])]
        return sb.xs[0] if name == "xs0" else getattr(sb, name)

    # ---- one iteration ----
    def step(self, tokens, *, timing: bool = False) -> dict:
        """One synchronous training iteration over the M microbatches; returns the loss.

        Ops are issued in the simulator's global order, each on its node's stream.  A node's op
        waits only for its own inputs: an NCCL receive (remote hop) or the producer's completion
        event followed by a D2D copy on the consumer's stream (local hop between nodes)."""
        host = tokens if isinstance(tokens, dict) else self._stage_inputs(tokens)
        self.step_count += 1
        s = self.stream
        ev, ev_lw = {}, {}
        t_iter0 = torch.cuda.Event(enable_timing=True)
        t_iter1 = torch.cuda.Event(enable_timing=True)
        pending: dict = {}
        sends: list = []
        streams = list(dict.fromkeys(self.nstream[v] for v in self.my_nodes))
        with torch.cuda.device(self.dev):
            s.wait_stream(torch.cuda.current_stream(self.dev))
            t_iter0.record(s)
            with torch.cuda.stream(s):
                if self.keep_grads:
                    for ps in self.psets.values():
                        ps.g.zero_()
                    for gl in self.extra_grads.values():
                        for g in gl:
                            g.zero_()
                if self.world > 1:
                    self.mb_loss.zero_()   # summed over ranks; every slot is rewritten on one rank
            for cs in streams:
                if cs is not s:
                    cs.wait_stream(s)
            executed = []
            for idx, op in enumerate(self.ops):
                v, mb = op.node, op.mb
                mine = self.placement[v] == self.rank
                out = None
                if mine:
                    sv = self.nstream[v]
                    key = self._key(op)
                    sb = self.slots[(v, key[2])]
                    if op.kind == F and op.pos == 0:
                        # the slot keeps ids / targets / grouping until this microbatch's L and B
                        # ops at the origin (same node, same slot, same stream).  The embed needs
                        # only ids: split them here, sort for the embedding backward on the prep
                        # stream (joined before the B op at the origin)
                        _h2d(sb.tok, host["tokens"][mb], sv)
                        native.token_prep(sb.tok, sb.ids, sb.targets, None, None, None, None, b=self.b, T=self.T,
                                          stream=sv)
                        staged = torch.cuda.Event()
                        staged.record(sv)
                        self.prep_stream.wait_event(staged)
                        native.token_prep(sb.tok, None, None, sb.perm, sb.seg_start, sb.seg_id, sb.n_seg, b=self.b,
                                          T=self.T, stream=self.prep_stream)
                        grouped = torch.cuda.Event()
                        grouped.record(self.prep_stream)
                        self._prep_done[(v, key[2])] = grouped
                    if op.kind == B and op.pos == 0:
                        sv.wait_event(self._prep_done.pop((v, key[2])))
                    w = pending.pop((op.kind, v, op.agent, op.wave), None)
                    if w is not None:
                        if w[0] == "nccl":
                            with torch.cuda.stream(sv):
                                w[1].wait()        # input arrived from another rank
                        elif w[0] == "peer":       # pushed by another rank into this slot
                            native.hop_wait(w[1], w[2], stream=sv)
                        else:                      # local hop from another node's stream
                            _, src, src_ev, dst = w
                            sv.wait_event(src_ev)
                            native.hop(dst, self.dev.index, src, self.dev.index, src.numel() * src.element_size(),
                                       stream=sv)
                    if timing:
                        e0 = torch.cuda.Event(enable_timing=True)
                        e0.record(sv)
                    if self.use_graphs:
                        with torch.cuda.stream(sv):
                            self._graphs[key].replay()   # replays on the current stream
                        out = self._outs[key]
                    else:
                        out = self._run_op(op.kind, v, key[2], sv)
                    if timing:
                        e1 = torch.cuda.Event(enable_timing=True)
                        e1.record(sv)
                        ev[idx] = (e0, e1)
                    executed.append((idx, op.kind, v, op.agent, op.wave))
                    if op.kind == L:
                        with torch.cuda.stream(sv):
                            self.mb_loss[mb:mb + 1].copy_(sb.loss, non_blocking=True)
                hop = self.hops[idx]
                if hop is not None:
                    self._issue_hop(idx, op, hop, out, mine, pending, sends)
                for st in self._ar_after.get(idx, ()):
                    self._issue_allreduce(st, self.stream)
                if mine and op.kind == L:  # the head wgrad, after the returned gradient left
                    sv = self.nstream[v]
                    lw = (LW, v, self._key(op)[2])
                    if self.use_graphs:
                        with torch.cuda.stream(sv):
                            self._graphs[lw].replay()
                    else:
                        self._run_op(LW, v, lw[2], sv)
                    if timing:
                        e1 = torch.cuda.Event(enable_timing=True)
                        e1.record(sv)
                        ev_lw[idx] = e1
            for cs in streams:
                if cs is not s:
                    s.wait_stream(cs)
            s.wait_stream(self.prep_stream)
            self._finish_step(sends)
            t_iter1.record(s)
            torch.cuda.current_stream(self.dev).wait_stream(s)
            if self.world > 1:
                import torch.distributed as dist

                dist.all_reduce(self.mb_loss)
            loss = float(self.mb_loss.sum().item()) / self.M
        out = {"loss": loss, "executed": executed}
        if timing:
            torch.cuda.synchronize(self.dev)
            out["iter_ms"] = t_iter0.elapsed_time(t_iter1)
            out["op_times"] = {i: (t_iter0.elapsed_time(a), t_iter0.elapsed_time(b_)) for i, (a, b_) in ev.items()}
            # an L op's head weight gradient (issued after the returned gradient left)
            out["lw_end"] = {i: t_iter0.elapsed_time(e) for i, e in ev_lw.items()}
        return out

    def _issue_hop(self, idx, op, hop, out, mine, pending, sends):
        """The path hop that follows op ``idx``: a local copy (or its deferred form), an NCCL send
        from a slot-owned buffer, or the matching receive."""
        v = op.node
        nv, name, _, dst_rank, consumer = hop
        dst_mine = dst_rank == self.rank
        if mine and dst_mine:
            buf = self._dst_buffer(op, nv, name)
            sv = self.nstream[v]
            if self.nstream[nv] is sv:
                native.hop(buf, self.dev.index, out, self.dev.index, out.numel() * out.element_size(),
                           stream=sv)
            else:
                # copied on the consumer's stream right before the consumer op: the
                # destination slot is then free (the consumer node's earlier ops are ahead
                # of it on that stream) and the source is slot-owned until the agent's next
                # wave, which causally follows the consumer
                done = torch.cuda.Event()
                done.record(sv)
                pending[(consumer, nv, op.agent, op.wave)] = ("local", out, done, buf)
        elif mine:
            import torch.distributed as dist

            # the source is slot-owned (F: last residual buffer, B: gout, L: dret) and is
            # rewritten only by this agent's next wave, which causally follows this send's
            # completion: drain it on the send stream without stalling compute
            ev_out = torch.cuda.Event()
            ev_out.record(self.nstream[v])
            ss = self.nsend[v]
            ss.wait_event(ev_out)
            if self.hop_transport == "peer":
                # push straight into the consumer's slot on the peer GPU (static slots: its last
                # reader causally precedes this producer), then release the slot's arrival flag
                k = (nv, self.slot_of[(op.agent, nv)], name)
                self._push(self._peer_addr[k], out, self._peer_flag[k], ss)
                sends.append((None, ss))
            else:
                with torch.cuda.stream(ss):
                    sends.append((dist.isend(out, dst_rank, group=self._pair[dst_rank]), ss))
        elif dst_mine:
            import torch.distributed as dist

            if self.hop_transport == "peer":
                k = (nv, self.slot_of[(op.agent, nv)], name)
                self._flag_expect[k] += self.hop_inc
                pending[(consumer, nv, op.agent, op.wave)] = ("peer", self._flag_local[k], self._flag_expect[k])
                return
            buf = self._dst_buffer(op, nv, name)
            # the destination slot was last read by this agent's previous wave on the
            # consumer node, whose ops so far are all on that node's stream
            rs = self.nrecv[nv]
            rs.wait_stream(self.nstream[nv])
            with torch.cuda.stream(rs):
                w = dist.irecv(buf, self.placement[v], group=self._pair[self.placement[v]])
            pending[(consumer, nv, op.agent, op.wave)] = ("nccl", w)

    def _issue_allreduce(self, st: int, after):
        """Sum stage st's flat fp32 gradient over the ranks holding it (spx_allreduce on the
        stage's libspx communicator) on the stage's own stream, once ``after`` (the stream of the
        rank's last op of the stage) has produced it."""
        cs = self._ar_stream[st]
        # every stream that ran an op of the stage on this rank (per-node streams) has finished it
        for sv in dict.fromkeys([after] + [self.nstream[v] for v in self.my_nodes if self.node_stage[v] == st]):
            ev = torch.cuda.Event()
            ev.record(sv)
            cs.wait_event(ev)
        ps = self.psets[st]
        for g in self.extra_grads[st]:  # co-resident replicas first, in node order
            native.add_f32(ps.g, g, ps.lay.numel, clear=not self.keep_grads, stream=cs)
        native.allreduce(self._groups[st], ps.g, ps.lay.numel, stream=cs)

    def _finish_step(self, sends):
        """Drain the hop sends, then the replica sum / clip / AdamW on the rank's main stream."""
        s = self.stream
        if sends:
            with torch.cuda.stream(s):
                for w, _ in sends:
                    if w is not None:
                        w.wait()
            for ss in dict.fromkeys(ss for _, ss in sends):
                s.wait_stream(ss)
        self.optimizer_step()

    # ---- optimizer ----
    def launches_per_step(self) -> int:
        """libspx kernel launches in one iteration on this rank (graph contents + optimizer)."""
        if not self.use_graphs:
            raise ValidationError("launch accounting needs use_graphs=True")
        opt = 2 * len(self.psets) + 1 + len(self.psets) + sum(len(gl) for gl in self.extra_grads.values())
        # (+ torch fills when keep_grads: not libspx launches)
        mine = [self._key(op) for op in self.ops if self.placement[op.node] == self.rank]
        prep = 2 * sum(1 for op in self.ops if op.kind == F and op.pos == 0 and self.placement[op.node] == self.rank)
        return prep + sum(self._graph_launches[k] + (self._graph_launches[(LW,) + k[1:]] if k[0] == L else 0)
                   for k in mine) + opt

    def gemm_counts_per_step(self) -> dict:
        """GEMM key -> launches per iteration on this rank (needs native.record_gemms at setup)."""
        out: dict = {}
        for op in self.ops:
            if self.placement[op.node] == self.rank:
                k = self._key(op)
                keys = [k] + ([(LW,) + k[1:]] if k[0] == L else [])
                for gk in keys:
                    for key in self._graph_gemms.get(gk, []):
                        out[key] = out.get(key, 0) + 1
        return out

    def optimizer_step(self):
        """Replica all-reduce (NCCL, only for stages replicated across ranks), global-norm clip and
        AdamW, all enqueued on the compute stream — no host synchronisation."""
        o = self.optim
        s = self.stream
        with torch.cuda.stream(s):
            for st, gl in self.extra_grads.items():  # co-resident replicas, in node order
                if st in self._groups:
                    continue                          # merged before its all-reduce
                for g in gl:
                    native.add_f32(self.psets[st].g, g, self.psets[st].lay.numel, clear=not self.keep_grads, stream=s)
            for st in self._groups:  # replica all-reduces, issued during the step (_issue_allreduce)
                s.wait_stream(self._ar_stream[st])
            self._sumsq.zero_()
            for st in self.my_stages:
                # each stage counted once: its lowest hosting rank contributes the squared norm
                if self.stage_ranks[st][0] == self.rank:
                    ps = self.psets[st]
                    native.sumsq(ps.g, ps.lay.numel, self._sumsq_ws, self._sumsq[st:st + 1], stream=s)
            if self.world > 1:
                import torch.distributed as dist

                dist.all_reduce(self._sumsq)
            native.clip_scale(self._sumsq, self.assignment.s, o.max_grad_norm, self._clip, self._norm, stream=s)
            for st in self.my_stages:
                ps = self.psets[st]
                native.adamw(ps.p32, ps.g, ps.m, ps.v, ps.pbf, n=ps.lay.numel, n_decay=ps.lay.n_decay, lr=o.lr,
                             beta1=o.beta1, beta2=o.beta2, eps=o.eps, weight_decay=o.weight_decay,
                             step=self.step_count, grad_scale=self._clip, clear_grad=not self.keep_grads, stream=s)

    # ---- inspection (tests) ----
    def grads(self) -> dict[int, dict[str, torch.Tensor]]:
        """Canonical fp32 gradients of the last iteration (post replica-sum, pre-clip) for the
        stages hosted on this rank (needs keep_grads=True: otherwise AdamW cleared them)."""
        if not self.keep_grads:
            raise ValidationError("grads() needs Trainer(keep_grads=True): the optimizer clears consumed gradients")
        torch.cuda.synchronize(self.dev)
        return {st: unpack_stage(self.cfg, self.layouts[st], self.psets[st].g) for st in self.my_stages}

    def params(self) -> dict[int, dict[str, torch.Tensor]]:
        torch.cuda.synchronize(self.dev)
        return {st: unpack_stage(self.cfg, self.layouts[st], self.psets[st].p32) for st in self.my_stages}

    # ---- skip-robust inference (§5) ----
    def eval_loss(self, tokens: torch.Tensor, stages: list[int], partial: dict | None = None) -> float:
        """Token-mean cross-entropy of one microbatch (tokens [b, T+1]) run forward through
        ``stages`` (stage 0 first; any subset / order, as in training paths) and back to the
        loss at the origin, with the current weights -- no gradients.  ``partial`` maps a stage
        to the number of its first layers to execute (the paper's partial stage skips).  Uses
        the first hosted node of each stage and its slot 0, so call it between iterations.  One
        process holding every stage (world == 1)."""
        if self.world != 1:
            raise ValidationError("eval_loss runs on a single process that hosts every stage")
        if not stages or stages[0] != 0:
            raise ValidationError(f"an inference path starts at stage 0, got {stages}")
        if tokens.shape != (self.b, self.T + 1):
            raise ValidationError(f"tokens shape {tuple(tokens.shape)} != ({self.b}, {self.T + 1})")
        partial = partial or {}
        node_of = {}
        for v in self.my_nodes:
            node_of.setdefault(self.node_stage[v], v)
        s = self.stream
        with torch.cuda.device(self.dev), torch.cuda.stream(s):
            s.wait_stream(torch.cuda.current_stream(self.dev))
            for v in self.my_nodes:
                s.wait_stream(self.nstream[v])
            origin = self.slots[(node_of[0], 0)]
            origin.ids.copy_(tokens[:, :-1].reshape(-1).to(torch.int32), non_blocking=True)
            origin.targets.copy_(tokens[:, 1:].reshape(-1).to(torch.int32), non_blocking=True)
            x = None
            for st in stages:
                v = node_of[st]
                sb = self.slots[(v, 0)]
                if x is not None:
                    sb.xs[0].copy_(x)
                x = self.prog.fwd(self.nparams[v], sb, self.nscratch[v], st == 0, s, partial.get(st))
            origin.ret.copy_(x)
            v0 = node_of[0]
            self.prog.loss_fwd(self.nparams[v0], origin, self.nscratch[v0], s)
            loss = float(origin.loss.item())
        return loss

    def skip_eval(self, tokens: torch.Tensor, skip_rate: float, seed: int = 0) -> float:
        """Perplexity with ``skip_rate`` of the stages dropped at random per microbatch, never
        stage 0; when the rate does not divide into whole stages the last dropped
        stage is half-executed (its first half of layers).  tokens [M, b, T+1]."""
        s_ = self.assignment.s
        gen = torch.Generator().manual_seed(seed)
        drop = skip_rate * s_
        whole = int(math.floor(drop + 1e-9))
        half = drop - whole > 1e-9
        losses = []
        for mb in range(tokens.shape[0]):
            order = (torch.randperm(s_ - 1, generator=gen) + 1).tolist()
            dropped, partial_st = set(order[:whole]), (order[whole] if half and whole < s_ - 1 else None)
            stages = [st for st in range(s_) if st not in dropped]
            partial = {partial_st: max(1, self.split[partial_st] // 2)} if partial_st is not None else None
            losses.append(self.eval_loss(tokens[mb], stages, partial))
        return math.exp(sum(losses) / len(losses))

    def grad_norm(self) -> float:
        torch.cuda.synchronize(self.dev)
        return float(self._norm.item())

    def make_report(self, res: dict) -> ExecReport:
        """ExecReport (SimReport fields measured on this rank's device) from step(timing=True)."""
        n = self.topology.n
        busy = [0.0] * n
        order: dict[int, list] = {}
        trace, start_f0 = [], {}
        e2e = [0.0] * self.M
        for idx, kind, v, agent, wave in res["executed"]:
            t0, t1 = res["op_times"][idx]
            busy[v] += res.get("lw_end", {}).get(idx, t1) - t0
            order.setdefault(v, []).append((kind, agent, wave))
            dirn = {"F": "fwd", "L": "loss", "B": "bwd"}[kind]
            trace.append((t0, v, "start", agent, wave, dirn))
            trace.append((t1, v, "end", agent, wave, dirn))
            op = self.ops[idx]
            if kind == F and op.pos == 0:
                start_f0[op.mb] = t0
            if kind == B and op.pos == 0:
                e2e[op.mb] = t1 - start_f0[op.mb]
        # collision wait = sum over ops of (start - ready) as in the simulator, where
        # ready is the end of the op that produced the input (F at the origin: the end of the
        # agent's previous wave, or the iteration start).  Exact for producers on this rank (all
        # ops at one GPU); ops fed from another rank are left out (no common clock across GPUs).
        wait, counted = 0.0, 0
        key = {(op.agent, op.wave, op.kind, op.pos): i for i, op in enumerate(self.ops)}
        for idx, kind, v, agent, wave in res["executed"]:
            op = self.ops[idx]
            last = len(self.paths[agent]) - 1
            if kind == F:
                prod = key.get((agent, wave, F, op.pos - 1)) if op.pos > 0 else key.get((agent, wave - 1, B, 0))
            elif kind == L:
                prod = key[(agent, wave, F, last)]
            else:
                prod = key[(agent, wave, L, 0)] if op.pos == last else key[(agent, wave, B, op.pos + 1)]
            if prod is None:
                ready = 0.0
            elif prod in res["op_times"]:
                ready = res["op_times"][prod][1]
            else:
                continue
            wait += max(0.0, res["op_times"][idx][0] - ready)
            counted += 1
        self.collision_wait_ops = counted
        mk = res["iter_ms"]
        return ExecReport(iteration_makespan=mk, microbatch_e2e=e2e, total_collision_wait=wait, node_busy=busy,
                          node_idle=[mk - x for x in busy], loss=res["loss"], mb_loss=self.mb_loss.tolist(),
                          grad_norm=self.grad_norm(), node_order=order, trace=trace)


def _h2d(dst: torch.Tensor, src: torch.Tensor, stream) -> None:
    with torch.cuda.stream(stream):
        dst.copy_(src, non_blocking=True)


def execute(schedule: Schedule, topology: Topology, sim_config: SimConfig, model_cfg: ModelConfig, placement,
            tokens: torch.Tensor, *, assignment, b: int, split=None, seed: int = 0, steps: int = 1,
            use_graphs: bool = True, rank: int = 0, world: int = 1) -> ExecReport:
    """Drop-in for ``simulate``: same schedule / topology / sim_config, plus the model,
    a node->rank placement and the tokens; runs ``steps`` real iterations and returns the last
    one's measured report (losses included)."""
    tr = Trainer(schedule, topology, sim_config, model_cfg, assignment, b=b, T=tokens.shape[-1] - 1, split=split,
                 placement=placement, seed=seed, use_graphs=use_graphs, rank=rank, world=world)
    res = None
    for _ in range(steps):
        res = tr.step(tokens, timing=True)
    return tr.make_report(res)
