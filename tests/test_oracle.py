"""Pinning the CPU oracle itself (tests/ only): its attention equals torch's SDPA, its optimizer
step equals torch.optim.AdamW + clip_grad_norm_, its skip semantics are what PAPER.md describes,
and the product's HBM parameter layout round-trips the oracle's canonical tensors."""

import math

import torch

from oracle import train_ref
from paper_2502_19913_b200.model import (init_params, model_config, pack_stage, split_gate_up, stage_layout,
                                         synthetic_tokens, unpack_stage)


def tiny():
    return model_config("llama-50m", n_layers=4, vocab=512, context=64)


def test_attention_matches_sdpa():
    torch.manual_seed(0)
    cfg = tiny()
    p = init_params(cfg, [2, 2])[0]
    x = torch.randn(2, 64, cfg.d)
    cos, sin = train_ref.rope_tables(64, cfg.head_dim, cfg.rope_theta)
    # reproduce the attention block with SDPA
    h = train_ref.rms_norm(x, p["l0.attn_norm"], cfg.eps)
    q = train_ref.apply_rope((h @ p["l0.wq"].t()).view(2, 64, 6, 48), cos, sin).transpose(1, 2)
    k = train_ref.apply_rope((h @ p["l0.wk"].t()).view(2, 64, 6, 48), cos, sin).transpose(1, 2)
    v = (h @ p["l0.wv"].t()).view(2, 64, 6, 48).transpose(1, 2)
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    x1 = x + o.transpose(1, 2).reshape(2, 64, -1) @ p["l0.wo"].t()
    h2 = train_ref.rms_norm(x1, p["l0.mlp_norm"], cfg.eps)
    ref = x1 + (torch.nn.functional.silu(h2 @ p["l0.w_gate"].t()) * (h2 @ p["l0.w_up"].t())) @ p["l0.w_down"].t()
    got = train_ref.decoder_layer(x, p, 0, cfg, cos, sin)
    assert torch.allclose(got, ref, atol=1e-5, rtol=1e-4)


def test_optimizer_matches_torch_adamw():
    cfg = tiny()
    split = [2, 2]
    params = init_params(cfg, split, seed=3)
    tokens = synthetic_tokens(cfg, 2, 1, 64, seed=5)
    out = train_ref.iteration(cfg, split, params, [(0, 1), (0,)], tokens, max_norm=0.5)
    leaves = [{k: v.clone().requires_grad_() for k, v in p.items()} for p in params]
    groups = [{"params": [t for p in leaves for k, t in p.items() if not k.endswith("norm")], "weight_decay": 0.1},
              {"params": [t for p in leaves for k, t in p.items() if k.endswith("norm")], "weight_decay": 0.0}]
    opt = torch.optim.AdamW(groups, lr=3e-4, betas=(0.9, 0.95), eps=1e-8)
    for p, g in zip(leaves, out["grads"]):
        for k in p:
            p[k].grad = g[k].clone()
    torch.nn.utils.clip_grad_norm_([t for p in leaves for t in p.values()], 0.5)
    opt.step()
    for p, q in zip(leaves, out["params"]):
        for k in p:
            assert torch.allclose(p[k].detach(), q[k], atol=1e-7, rtol=0), k


def test_skipped_stage_gets_no_gradient_and_swap_changes_order():
    cfg = tiny()
    split = [1, 1, 1, 1]
    params = init_params(cfg, split, seed=1)
    tokens = synthetic_tokens(cfg, 1, 1, 64)
    out = train_ref.iteration(cfg, split, params, [(0, 2, 3)], tokens, update=False)
    assert all(float(g.abs().sum()) == 0.0 for g in out["grads"][1].values())   # stage 1 skipped
    a = train_ref.iteration(cfg, split, params, [(0, 2, 1)], tokens, update=False)["loss"]
    b = train_ref.iteration(cfg, split, params, [(0, 1, 2)], tokens, update=False)["loss"]
    assert a != b                                                                # swap = reordered stages


def test_initial_loss_near_log_vocab():
    cfg = tiny()
    params = init_params(cfg, [2, 2])
    tokens = synthetic_tokens(cfg, 2, 2, 64)
    out = train_ref.iteration(cfg, [2, 2], params, [(0, 1), (0, 1)], tokens, update=False)
    assert abs(out["loss"] - math.log(cfg.vocab)) < 0.2


def test_hbm_layout_roundtrip():
    cfg = tiny()
    split = [2, 2]
    params = init_params(cfg, split, seed=2)
    for st in range(2):
        lay = stage_layout(cfg, st, split)
        flat = pack_stage(cfg, lay, params[st])
        back = unpack_stage(cfg, lay, flat)
        assert set(back) == set(params[st])
        for k in back:
            assert torch.equal(back[k], params[st][k]), k
        # matrices before norms: weight decay prefix covers exactly the matrices
        for name, slot in lay.slots.items():
            assert (slot.offset < lay.n_decay) == (not name.endswith("norm"))
    wg, wu = split_gate_up(pack_stage(cfg, stage_layout(cfg, 0, split), params[0])[
        stage_layout(cfg, 0, split).slots["l0.wgu"].offset:][: 2 * cfg.ffn * cfg.d].view(2 * cfg.ffn, cfg.d))
    assert torch.equal(wg, params[0]["l0.w_gate"]) and torch.equal(wu, params[0]["l0.w_up"])
