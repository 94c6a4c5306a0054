"""ORACLE — test infrastructure only.  CPU fp32 restatement of one SkipPipe training iteration.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference / cpu_baseline leg may
import this module; the product path (``paper_2502_19913_b200``) never does.

What it restates.  The reference ships no training code (SPEC.md:12 puts "actual LLM training
and gradient math" out of scope), so no *reference* vector can pin losses or gradients.  The
restatement is instead pinned to an independent published LLaMA implementation: Hugging Face
transformers.LlamaForCausalLM (fp64) reproduces its loss to 1e-9 and every gradient tensor to
1e-6 relative on full, skipped and swapped stage paths, MHA and GQA (oracle/gen_hf_golden.py ->
tests/golden/hf_llama_golden.json, tests/test_oracle_hf.py).

* LLaMA decoder (Table 4 at :495-499): RMSNorm → QKV (+RoPE, rotate-half) →
  causal softmax attention (GQA by head repetition) → O proj + residual → RMSNorm → SwiGLU MLP
  + residual.  S₀ additionally holds the token embedding, the final RMSNorm and the untied
  de-embedding head; the loss is computed on S₀ when the microbatch returns.
* Partial / reordered pipeline: microbatch ``mb`` of wave ``w`` on
  agent ``a`` runs the stages of that agent's first-wave path in path order (skipped stages are
  not executed, a swap runs two stages out of order), forward then backward.
* Gradient accumulation over the M microbatches of an iteration with the loss
  normalised as mean over microbatches of the per-token mean cross-entropy; stage replicas'
  gradients are summed (DP) — mathematically one gradient per stage.
* Synchronous update: global-norm clip 1.0 then AdamW, lr 3e-4,
  betas (0.9, 0.95), eps 1e-8, weight decay 0.1 on matrices/embeddings only.
"""

from __future__ import annotations

import math

import torch

F32 = torch.float32


def rope_tables(T: int, hd: int, theta: float, device=None):
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    ang = torch.arange(T, dtype=torch.float64)[:, None] * inv[None, :]
    return ang.cos().to(F32).to(device), ang.sin().to(F32).to(device)


def rms_norm(x, g, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def apply_rope(x, cos, sin):
    # x [b, T, h, hd]; rotate-half convention
    half = x.shape[-1] // 2
    c = cos[None, :, None, :]
    s = sin[None, :, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def decoder_layer(x, p, i, cfg, cos, sin):
    b, T, d = x.shape
    H, Hkv, hd = cfg.n_heads, cfg.n_kv_heads, cfg.d // cfg.n_heads
    h = rms_norm(x, p[f"l{i}.attn_norm"], cfg.eps)
    q = (h @ p[f"l{i}.wq"].t()).view(b, T, H, hd)
    k = (h @ p[f"l{i}.wk"].t()).view(b, T, Hkv, hd)
    v = (h @ p[f"l{i}.wv"].t()).view(b, T, Hkv, hd)
    q, k = apply_rope(q, cos, sin), apply_rope(k, cos, sin)
    q, k, v = (t.permute(0, 2, 1, 3) for t in (q, k, v))
    rep = H // Hkv
    k = k.repeat_interleave(rep, dim=1)
    v = v.repeat_interleave(rep, dim=1)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
    mask = torch.ones(T, T, dtype=torch.bool, device=x.device).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    o = (torch.softmax(s, dim=-1) @ v).permute(0, 2, 1, 3).reshape(b, T, H * hd)
    x = x + o @ p[f"l{i}.wo"].t()
    h = rms_norm(x, p[f"l{i}.mlp_norm"], cfg.eps)
    gate = h @ p[f"l{i}.w_gate"].t()
    up = h @ p[f"l{i}.w_up"].t()
    return x + (torch.nn.functional.silu(gate) * up) @ p[f"l{i}.w_down"].t()


def stage_forward(x, p, n_layers, cfg, cos, sin):
    for i in range(n_layers):
        x = decoder_layer(x, p, i, cfg, cos, sin)
    return x


def microbatch_loss(tokens, stages, params, split, cfg, cos, sin):
    """tokens [b, T+1]; ``stages`` = the pipeline stages of this microbatch's path in order."""
    inp, tgt = tokens[:, :-1], tokens[:, 1:]
    x = params[0]["embed"][inp]
    for st in stages:
        x = stage_forward(x, params[st], split[st], cfg, cos, sin)
    x = rms_norm(x, params[0]["final_norm"], cfg.eps)
    logits = x @ params[0]["head"].t()
    return torch.nn.functional.cross_entropy(logits.reshape(-1, cfg.vocab), tgt.reshape(-1))


def is_decayed(name: str) -> bool:
    return not name.endswith("norm")


def iteration(cfg, split, params, mb_stages, tokens, opt_state=None, *, lr=3e-4, betas=(0.9, 0.95), eps=1e-8,
              weight_decay=0.1, max_norm=1.0, step=1, update=True, threads=None, device=None):
    """One synchronous iteration.

    params: list (per stage) of dicts of canonical fp32 tensors (not modified).
    mb_stages: list over microbatches of stage sequences (len M).
    tokens: int64 [M, b, T+1].
    device: where the fp32 arithmetic runs (default: the CPU).  Tests at the C2-C4 shapes run
    the same fp32 restatement on the GPU with TF32 off, as a checker (it is not the product).
    Returns dict(loss, mb_loss, grads, grad_norm, params (updated), opt_state), on ``device``.
    """
    if threads:
        torch.set_num_threads(threads)
    M = len(mb_stages)
    T = tokens.shape[-1] - 1
    tokens = tokens.to(device)
    cos, sin = rope_tables(T, cfg.d // cfg.n_heads, cfg.rope_theta, device)
    leaves = [{k: v.detach().to(device, F32).clone().requires_grad_(True) for k, v in p.items()} for p in params]
    if opt_state is not None:
        opt_state = [{k: (m.to(device), v.to(device)) for k, (m, v) in s.items()} for s in opt_state]
    params = [{k: v.detach().to(device, F32) for k, v in p.items()} for p in params]
    mb_loss = []
    for mb in range(M):
        loss = microbatch_loss(tokens[mb], mb_stages[mb], leaves, split, cfg, cos, sin)
        (loss / M).backward()
        mb_loss.append(float(loss.detach()))
    grads = [{k: (v.grad if v.grad is not None else torch.zeros_like(v)) for k, v in p.items()} for p in leaves]
    total = math.sqrt(sum(float(g.double().pow(2).sum()) for gs in grads for g in gs.values()))
    out = {"loss": sum(mb_loss) / M, "mb_loss": mb_loss, "grads": grads, "grad_norm": total}
    if not update:
        return out
    clip = min(1.0, max_norm / (total + 1e-6))
    st = opt_state or [{k: (torch.zeros_like(v), torch.zeros_like(v)) for k, v in p.items()} for p in params]
    b1, b2 = betas
    bc1, bc2 = 1 - b1**step, 1 - b2**step
    new_params, new_state = [], []
    for p, gs, s in zip(params, grads, st):
        np_, ns = {}, {}
        for k, w in p.items():
            g = gs[k] * clip
            m, v = s[k]
            m = b1 * m + (1 - b1) * g
            v = b2 * v + (1 - b2) * g * g
            w = w.clone()
            if is_decayed(k):
                w = w * (1 - lr * weight_decay)
            w = w - (lr / bc1) * m / (v.sqrt() / math.sqrt(bc2) + eps)
            np_[k], ns[k] = w, (m, v)
        new_params.append(np_)
        new_state.append(ns)
    out.update(params=new_params, opt_state=new_state)
    return out


def mb_stage_sequences(paths_stages: dict, agents_sorted: list, M: int) -> list:
    """Microbatch mb = wave·|P| + index(agent) runs its agent's first-wave stage path
    (waves reuse first-wave paths)."""
    P = len(agents_sorted)
    return [tuple(paths_stages[agents_sorted[mb % P]]) for mb in range(M)]
