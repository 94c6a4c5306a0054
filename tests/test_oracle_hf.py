"""Pin of the oracle's training math (oracle/train_ref.py) to an independent published LLaMA
implementation: Hugging Face transformers.LlamaForCausalLM (fp64, eager attention).  The
reference itself has no training code, so this is the strongest available anchor:

* golden fixture tests/golden/hf_llama_golden.json (made by oracle/gen_hf_golden.py): per
  SkipPipe stage path -- full, skipped and swapped stage sequences, MHA and GQA models -- the HF
  loss and every gradient tensor's norm and sum; the oracle (run in fp64) must match (loss 1e-9, gradients 1e-6
  relative; the residual is the fp32 RoPE tables of the two implementations);
* live cross-check against transformers when it is importable (it is in this image).
"""

import json
import os

import pytest
import torch

from oracle import train_ref
from paper_2502_19913_b200.model import init_params, model_config, synthetic_tokens

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "hf_llama_golden.json")


def _oracle_path(cfg, params, split, stages, tokens):
    p64 = [{k: v.double().clone().requires_grad_(True) for k, v in p.items()} for p in params]
    T = tokens.shape[-1] - 1
    cos, sin = train_ref.rope_tables(T, cfg.head_dim, cfg.rope_theta)
    loss = train_ref.microbatch_loss(tokens, stages, p64, split, cfg, cos.double(), sin.double())
    loss.backward()
    g = {}
    for st in stages:
        for k, v in p64[st].items():
            if k.startswith("l") or st == 0:
                if v.grad is not None:
                    g[f"{st}:{k}"] = v.grad
    return float(loss), g


def _cases():
    with open(GOLD) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["name"])
def test_oracle_matches_hf_golden(case):
    cfg = model_config("llama-50m", **case["model"])
    params = init_params(cfg, case["split"], seed=case["param_seed"])
    tokens = synthetic_tokens(cfg, len(case["paths"]), case["b"], case["T"], seed=case["token_seed"])
    for k, row in enumerate(case["paths"]):
        loss, g = _oracle_path(cfg, params, case["split"], row["stages"], tokens[k])
        assert abs(loss - row["loss"]) <= 1e-9 * abs(row["loss"]), (row["stages"], loss, row["loss"])
        assert set(g) == set(row["grad_norm"]), row["stages"]
        for key, ref in row["grad_norm"].items():
            got = float(g[key].norm())
            assert abs(got - ref) <= 1e-6 * max(ref, 1e-30), (row["stages"], key, got, ref)
            s = float(g[key].sum())
            assert abs(s - row["grad_sum"][key]) <= 1e-6 * max(ref, 1e-30) * g[key].numel() ** 0.5, (key, s)


def test_oracle_matches_hf_live():
    pytest.importorskip("transformers")
    from oracle.gen_hf_golden import hf_path_loss_grads

    cfg = model_config("llama-50m", d=64, n_heads=4, n_kv_heads=2, ffn=128, vocab=96, n_layers=3)
    split = [1, 1, 1]
    params = init_params(cfg, split, seed=3)
    tokens = synthetic_tokens(cfg, 1, 2, 16, seed=11)[0]
    for stages in ([0, 1, 2], [0, 2, 1], [0, 2]):
        ref_loss, ref_g = hf_path_loss_grads(cfg, params, split, stages, tokens)
        loss, g = _oracle_path(cfg, params, split, stages, tokens)
        assert abs(loss - ref_loss) <= 1e-9 * ref_loss
        for (st, name), t in ref_g.items():
            d = float((g[f"{st}:{name}"] - t).norm())
            assert d <= 1e-6 * float(t.norm()), (stages, st, name, d)
