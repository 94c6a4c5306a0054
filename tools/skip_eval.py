"""Skip-robust inference (§5, Table 2 protocol).

    python tools/skip_eval.py [--config C2] [--steps 3] [--rates 0,0.25,0.5]

Trains ``--steps`` SkipPipe iterations on the synthetic batch, then reports the perplexity of
the batch with the given fraction of stages dropped at random per microbatch (never stage 0;
a non-integral count half-executes one more stage), plus early exits (stage 0..j then the head).
With i.i.d. uniform synthetic tokens the absolute numbers only show the mechanism working (the
model memorises its one batch); the paper's Arxiv perplexities need real data.
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_19913_b200.configs import get_config  # noqa: E402
from paper_2502_19913_b200.executor import Trainer  # noqa: E402
from paper_2502_19913_b200.model import synthetic_tokens  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--rates", default="0,0.25,0.5")
    a = ap.parse_args()
    rc = get_config(a.config)
    tr = Trainer(rc.schedule(), rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split)
    tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T)
    host = tr._stage_inputs(tokens)
    for i in range(a.steps):
        print(f"train step {i}: loss {tr.step(host)['loss']:.4f}", flush=True)
    ev = tokens[: min(8, rc.M)]
    for r in (float(x) for x in a.rates.split(",")):
        print(f"inference skip rate {r:.2f}: perplexity {tr.skip_eval(ev, r, seed=0):.3f}", flush=True)
    for j in range(rc.s):
        ppl = math.exp(sum(tr.eval_loss(ev[m], list(range(j + 1))) for m in range(ev.shape[0])) / ev.shape[0])
        print(f"early exit after stage {j}: perplexity {ppl:.3f}", flush=True)


if __name__ == "__main__":
    main()
