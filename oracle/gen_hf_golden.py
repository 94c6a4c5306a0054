"""ORACLE pinning -- test infrastructure only.  Generates tests/golden/hf_llama_golden.json.

The reference ships no training math, so no reference vector can pin the loss or
gradients of oracle/train_ref.py.  The closest independent anchor is a published LLaMA
implementation: Hugging Face ``transformers.LlamaForCausalLM`` (transformers 5.5.0 in this image,
eager attention, fp64).  This script builds tiny models with the conventions the oracle restates
(RMSNorm, rotate-half RoPE, GQA, SwiGLU MLP, untied head), loads the oracle's
initial weights, runs microbatches along SkipPipe stage paths -- a path with skipped and swapped
stages is the same decoder stack with the visited stages' layers concatenated in path order
 -- and records HF's loss and per-tensor gradient norms and sums.

    python oracle/gen_hf_golden.py      # rewrites tests/golden/hf_llama_golden.json
"""

from __future__ import annotations

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "tests", "golden", "hf_llama_golden.json")

# (name, model overrides, layer split, paths (stage sequences), b, T)
CASES = [
    ("mha_4stage", dict(d=64, n_heads=4, n_kv_heads=4, ffn=256, vocab=128, n_layers=4), [1, 1, 1, 1],
     [[0, 1, 2, 3], [0, 2, 3], [0, 2, 1, 3], [0, 3, 1]], 2, 32),
    ("gqa_3stage", dict(d=96, n_heads=6, n_kv_heads=2, ffn=256, vocab=160, n_layers=6), [2, 2, 2],
     [[0, 1, 2], [0, 2], [0, 2, 1]], 2, 24),
]


def model_cfg(over):
    from paper_2502_19913_b200.model import model_config

    return model_config("llama-50m", **over)


def hf_path_model(cfg, params, split, stages):
    """LlamaForCausalLM whose decoder stack is the visited stages' layers in path order."""
    from transformers import LlamaConfig, LlamaForCausalLM

    n = sum(split[s] for s in stages)
    hc = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d, intermediate_size=cfg.ffn, num_hidden_layers=n,
                     num_attention_heads=cfg.n_heads, num_key_value_heads=cfg.n_kv_heads, rms_norm_eps=cfg.eps,
                     rope_theta=cfg.rope_theta, max_position_embeddings=4096, tie_word_embeddings=False,
                     attention_bias=False, mlp_bias=False, attn_implementation="eager")
    m = LlamaForCausalLM(hc).double()
    sd = {"model.embed_tokens.weight": params[0]["embed"], "model.norm.weight": params[0]["final_norm"],
          "lm_head.weight": params[0]["head"]}
    j = 0
    for s in stages:
        for i in range(split[s]):
            p = params[s]
            pre = f"model.layers.{j}."
            sd.update({pre + "input_layernorm.weight": p[f"l{i}.attn_norm"],
                       pre + "post_attention_layernorm.weight": p[f"l{i}.mlp_norm"],
                       pre + "self_attn.q_proj.weight": p[f"l{i}.wq"], pre + "self_attn.k_proj.weight": p[f"l{i}.wk"],
                       pre + "self_attn.v_proj.weight": p[f"l{i}.wv"], pre + "self_attn.o_proj.weight": p[f"l{i}.wo"],
                       pre + "mlp.gate_proj.weight": p[f"l{i}.w_gate"], pre + "mlp.up_proj.weight": p[f"l{i}.w_up"],
                       pre + "mlp.down_proj.weight": p[f"l{i}.w_down"]})
            j += 1
    m.load_state_dict({k: v.double() for k, v in sd.items()}, strict=True)
    return m


def hf_path_loss_grads(cfg, params, split, stages, tokens):
    """HF loss (token-mean CE of tokens[:, 1:] given tokens[:, :-1]) and gradients mapped back to
    the oracle's (stage, name) keys; a stage's layers appear once per path, so no summing."""
    m = hf_path_model(cfg, params, split, stages)
    logits = m(input_ids=tokens[:, :-1]).logits
    loss = torch.nn.functional.cross_entropy(logits.reshape(-1, cfg.vocab), tokens[:, 1:].reshape(-1))
    loss.backward()
    g = {(0, "embed"): m.model.embed_tokens.weight.grad, (0, "final_norm"): m.model.norm.weight.grad,
         (0, "head"): m.lm_head.weight.grad}
    names = {"input_layernorm": "attn_norm", "post_attention_layernorm": "mlp_norm", "self_attn.q_proj": "wq",
             "self_attn.k_proj": "wk", "self_attn.v_proj": "wv", "self_attn.o_proj": "wo", "mlp.gate_proj": "w_gate",
             "mlp.up_proj": "w_up", "mlp.down_proj": "w_down"}
    j = 0
    for s in stages:
        for i in range(split[s]):
            lay = m.model.layers[j]
            for hf, ours in names.items():
                mod = lay
                for part in hf.split("."):
                    mod = getattr(mod, part)
                g[(s, f"l{i}.{ours}")] = mod.weight.grad
            j += 1
    return float(loss), g


def main():
    from paper_2502_19913_b200.model import init_params, synthetic_tokens

    out = {"generator": "transformers.LlamaForCausalLM (eager attention, float64)",
           "transformers_version": __import__("transformers").__version__, "cases": []}
    for name, over, split, paths, b, T in CASES:
        cfg = model_cfg(over)
        params = init_params(cfg, split, seed=0)
        tokens = synthetic_tokens(cfg, len(paths), b, T, seed=7)
        rows = []
        for k, stages in enumerate(paths):
            loss, g = hf_path_loss_grads(cfg, params, split, stages, tokens[k])
            rows.append({"stages": stages, "loss": loss,
                         "grad_norm": {f"{s}:{n}": float(t.norm()) for (s, n), t in sorted(g.items())},
                         "grad_sum": {f"{s}:{n}": float(t.sum()) for (s, n), t in sorted(g.items())}})
        out["cases"].append({"name": name, "model": over, "split": split, "b": b, "T": T, "token_seed": 7,
                             "param_seed": 0, "paths": rows})
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
