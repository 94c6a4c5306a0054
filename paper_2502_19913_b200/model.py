"""LLaMA model shapes and the per-stage parameter layout in HBM.

``ModelConfig`` extends the reference's ``ModelPreset`` (topology.py:150-180, which only has
hidden dim, layers and context; Table 4 of PAPER.md:492-499 adds heads) with the fields a real
decoder needs (FFN width, vocab, KV heads, RoPE base) and an optional unequal layer split per
stage.  FFN = 256·⌈(8d/3)/256⌉ and vocab 32000 follow LLaMA conventions; the
8B preset uses LLaMA-3-8B dims (GQA 32q/8kv, FFN 14336, vocab 128256).

Parameter layout (one *parameter set* per pipeline stage): a single flat fp32 master buffer and
a flat bf16 working copy with identical offsets, so the optimizer is one kernel per set, the
replica all-reduce is one NCCL call per set, and every GEMM reads its weight straight out of the
bf16 buffer.  Decayed tensors (all matrices) come first, norm gains last, so AdamW applies
weight decay to the prefix [0, n_decay).  Each tensor starts on a 64-element boundary.

Canonical ("math") layout is the torch ``nn.Linear`` one ([out, in]); the HBM layout differs in
one place: the MLP gate and up projections are packed into one [2F, d] matrix with 128-row
interleaving (gate rows 0-127, up rows 0-127, gate rows 128-255, ...) so the SwiGLU epilogue of
the fused gate/up GEMM sees a gate column block and its up block in one 256-wide tile.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import torch

from .errors import ValidationError
from .topology import ModelPreset, get_preset

_ALIGN = 64


@dataclass(frozen=True)
class ModelConfig:
    name: str
    d: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    context: int
    eps: float = 1e-5
    rope_theta: float = 10000.0
    init_std: float = 0.02

    def __post_init__(self):
        if self.d % self.n_heads:
            raise ValidationError(f"hidden dim {self.d} not divisible by {self.n_heads} heads")
        if self.n_heads % self.n_kv_heads:
            raise ValidationError(f"{self.n_heads} heads not divisible by {self.n_kv_heads} kv heads")
        if self.ffn % 128:
            raise ValidationError(f"ffn {self.ffn} must be a multiple of 128 (SwiGLU tile interleave)")

    @property
    def head_dim(self) -> int:
        return self.d // self.n_heads

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def preset(self) -> ModelPreset:
        return ModelPreset(self.name, self.d, self.n_layers, self.context)

    def layer_params(self) -> int:
        hd = self.head_dim
        return (self.qkv_dim * self.d + self.d * self.n_heads * hd + 3 * self.d * self.ffn + 2 * self.d)

    def total_params(self) -> int:
        return self.n_layers * self.layer_params() + 2 * self.vocab * self.d + self.d

    def layer_flops_per_token(self, T: int) -> float:
        """Forward FLOPs per token of one decoder layer, causal attention counted at half."""
        lin = 2 * (self.qkv_dim * self.d + self.d * self.n_heads * self.head_dim + 3 * self.d * self.ffn)
        attn = 2 * 2 * T * self.n_heads * self.head_dim / 2
        return float(lin + attn)

    def head_flops_per_token(self) -> float:
        return 2.0 * self.d * self.vocab


def _ffn_rule(d: int) -> int:
    return 256 * math.ceil((8 * d / 3) / 256)


_HEADS = {"llama-50m": (6, 6), "llama-500m": (16, 16), "llama-1.5b": (16, 16), "llama-7b": (32, 32),
          "llama-8b": (32, 8)}
_OVERRIDES = {"llama-7b": {"ffn": 11008}, "llama-8b": {"ffn": 14336, "vocab": 128256, "rope_theta": 500000.0}}


def model_config(name: str, **overrides) -> ModelConfig:
    """LLaMA config for a reference preset name (topology.py:171-180) plus Table-4 heads."""
    p = get_preset(name)
    h, kv = _HEADS[name]
    kw = dict(name=name, d=p.hidden_dim, n_layers=p.n_layers, n_heads=h, n_kv_heads=kv, ffn=_ffn_rule(p.hidden_dim),
              vocab=32000, context=p.context)
    kw.update(_OVERRIDES.get(name, {}))
    kw.update(overrides)
    return ModelConfig(**kw)


def layer_split(cfg: ModelConfig, s: int, split: list[int] | None = None) -> list[int]:
    """Layers per pipeline stage; equal (ModelPreset.layers_per_stage, topology.py:165-168) unless
    an explicit split is given."""
    if split is None:
        return [cfg.preset.layers_per_stage(s)] * s
    if len(split) != s or sum(split) != cfg.n_layers or min(split) < 1:
        raise ValidationError(f"layer split {split} must have {s} positive entries summing to {cfg.n_layers}")
    return list(split)


# ---------------------------------------------------------------------------------------
# flat parameter-set layout
# ---------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Slot:
    name: str
    shape: tuple[int, ...]
    offset: int

    @property
    def numel(self) -> int:
        return math.prod(self.shape)


@dataclass
class StageLayout:
    stage: int
    first_layer: int
    n_layers: int
    has_embed: bool
    slots: dict[str, Slot] = field(default_factory=dict)
    n_decay: int = 0
    numel: int = 0

    def view(self, flat: torch.Tensor, name: str) -> torch.Tensor:
        s = self.slots[name]
        return flat[s.offset: s.offset + s.numel].view(s.shape)


def stage_layout(cfg: ModelConfig, stage: int, split: list[int]) -> StageLayout:
    first = sum(split[:stage])
    lay = StageLayout(stage=stage, first_layer=first, n_layers=split[stage], has_embed=(stage == 0))
    off = 0

    def add(name, shape):
        nonlocal off
        lay.slots[name] = Slot(name, tuple(shape), off)
        off += math.prod(shape)
        off = (off + _ALIGN - 1) // _ALIGN * _ALIGN

    d, hd = cfg.d, cfg.head_dim
    for i in range(lay.n_layers):
        add(f"l{i}.wqkv", (cfg.qkv_dim, d))
        add(f"l{i}.wo", (d, cfg.n_heads * hd))
        add(f"l{i}.wgu", (2 * cfg.ffn, d))
        add(f"l{i}.wdown", (d, cfg.ffn))
    if lay.has_embed:
        add("embed", (cfg.vocab, d))
        add("head", (cfg.vocab, d))
    lay.n_decay = off
    for i in range(lay.n_layers):
        add(f"l{i}.attn_norm", (d,))
        add(f"l{i}.mlp_norm", (d,))
    if lay.has_embed:
        add("final_norm", (d,))
    lay.numel = off
    return lay


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    F, d = w_gate.shape
    return torch.stack([w_gate.view(F // 128, 128, d), w_up.view(F // 128, 128, d)], dim=1).reshape(2 * F, d)


def split_gate_up(wgu: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    F2, d = wgu.shape
    v = wgu.view(F2 // 256, 2, 128, d)
    return v[:, 0].reshape(F2 // 2, d), v[:, 1].reshape(F2 // 2, d)


# ---------------------------------------------------------------------------------------
# initial weights (canonical math layout, fp32 on CPU, deterministic)
# ---------------------------------------------------------------------------------------
def init_params(cfg: ModelConfig, split: list[int], seed: int = 0) -> list[dict[str, torch.Tensor]]:
    """Per-stage dicts of canonical fp32 tensors: N(0, init_std) for matrices and embeddings,
    ones for RMSNorm gains.  Drawn in a fixed order from one CPU generator so the GPU executor
    and the CPU oracle start from bit-identical weights."""
    gen = torch.Generator().manual_seed(seed)
    d, hd = cfg.d, cfg.head_dim

    def normal(*shape):
        return torch.randn(*shape, generator=gen, dtype=torch.float32) * cfg.init_std

    out = []
    for st in range(len(split)):
        p: dict[str, torch.Tensor] = {}
        if st == 0:
            p["embed"] = normal(cfg.vocab, d)
        for i in range(split[st]):
            p[f"l{i}.attn_norm"] = torch.ones(d)
            p[f"l{i}.wq"] = normal(cfg.n_heads * hd, d)
            p[f"l{i}.wk"] = normal(cfg.n_kv_heads * hd, d)
            p[f"l{i}.wv"] = normal(cfg.n_kv_heads * hd, d)
            p[f"l{i}.wo"] = normal(d, cfg.n_heads * hd)
            p[f"l{i}.mlp_norm"] = torch.ones(d)
            p[f"l{i}.w_gate"] = normal(cfg.ffn, d)
            p[f"l{i}.w_up"] = normal(cfg.ffn, d)
            p[f"l{i}.w_down"] = normal(d, cfg.ffn)
        if st == 0:
            p["final_norm"] = torch.ones(d)
            p["head"] = normal(cfg.vocab, d)
        out.append(p)
    return out


def pack_stage(cfg: ModelConfig, lay: StageLayout, params: dict[str, torch.Tensor]) -> torch.Tensor:
    """Canonical dict -> flat fp32 buffer in the HBM layout."""
    flat = torch.zeros(lay.numel, dtype=torch.float32)
    for i in range(lay.n_layers):
        lay.view(flat, f"l{i}.wqkv").copy_(torch.cat([params[f"l{i}.wq"], params[f"l{i}.wk"], params[f"l{i}.wv"]]))
        lay.view(flat, f"l{i}.wo").copy_(params[f"l{i}.wo"])
        lay.view(flat, f"l{i}.wgu").copy_(interleave_gate_up(params[f"l{i}.w_gate"], params[f"l{i}.w_up"]))
        lay.view(flat, f"l{i}.wdown").copy_(params[f"l{i}.w_down"])
        lay.view(flat, f"l{i}.attn_norm").copy_(params[f"l{i}.attn_norm"])
        lay.view(flat, f"l{i}.mlp_norm").copy_(params[f"l{i}.mlp_norm"])
    if lay.has_embed:
        for nm in ("embed", "head", "final_norm"):
            lay.view(flat, nm).copy_(params[nm])
    return flat


def unpack_stage(cfg: ModelConfig, lay: StageLayout, flat: torch.Tensor) -> dict[str, torch.Tensor]:
    """Flat buffer (params or grads, any device) -> canonical dict on CPU fp32."""
    flat = flat.detach().float().cpu()
    hd = cfg.head_dim
    qd, kd = cfg.n_heads * hd, cfg.n_kv_heads * hd
    out: dict[str, torch.Tensor] = {}
    for i in range(lay.n_layers):
        wqkv = lay.view(flat, f"l{i}.wqkv")
        out[f"l{i}.wq"], out[f"l{i}.wk"], out[f"l{i}.wv"] = wqkv[:qd], wqkv[qd:qd + kd], wqkv[qd + kd:]
        out[f"l{i}.wo"] = lay.view(flat, f"l{i}.wo")
        out[f"l{i}.w_gate"], out[f"l{i}.w_up"] = split_gate_up(lay.view(flat, f"l{i}.wgu"))
        out[f"l{i}.w_down"] = lay.view(flat, f"l{i}.wdown")
        out[f"l{i}.attn_norm"] = lay.view(flat, f"l{i}.attn_norm")
        out[f"l{i}.mlp_norm"] = lay.view(flat, f"l{i}.mlp_norm")
    if lay.has_embed:
        for nm in ("embed", "head", "final_norm"):
            out[nm] = lay.view(flat, nm)
    return {k: v.clone() for k, v in out.items()}


def rope_cos_sin(T: int, hd: int, theta: float) -> torch.Tensor:
    """[hd/2, T, 2] fp32 (cos, sin) of t·θ^(−2i/hd), computed in float64 then rounded.  Position-
    minor so the kernels' per-row lookups for one pair index are contiguous across a warp."""
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    ang = inv[:, None] * torch.arange(T, dtype=torch.float64)[None, :]
    return torch.stack([ang.cos(), ang.sin()], dim=-1).float().contiguous()


def synthetic_tokens(cfg: ModelConfig, M: int, b: int, T: int, seed: int = 1234) -> torch.Tensor:
    """i.i.d. uniform token ids [M, b, T+1] (inputs [..., :-1], targets [..., 1:]) — SURVEY.md §8(d)."""
    gen = torch.Generator().manual_seed(seed)
    return torch.randint(0, cfg.vocab, (M, b, T + 1), generator=gen, dtype=torch.int64)


def with_layers(cfg: ModelConfig, n_layers: int) -> ModelConfig:
    return replace(cfg, n_layers=n_layers)
