"""Run a short C2 iteration for profiling (ncu launch list / --set full captures).

    python tools/profile_step.py [--config C2] [--M 4] [--steps 2] [--eager]

--M overrides the microbatch count (one wave = |P| microbatches) so a launch list stays small.
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_19913_b200.configs import get_config  # noqa: E402
from paper_2502_19913_b200.executor import Trainer  # noqa: E402
from paper_2502_19913_b200.model import synthetic_tokens  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--M", type=int, default=4)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--eager", action="store_true")
    ap.add_argument("--gemm-log", default=None, help="write the GEMM call keys of the last step (eager) to this JSON")
    a = ap.parse_args()
    rc = get_config(a.config, M=a.M)
    tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T)
    tr = Trainer(rc.schedule(), rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split,
                 use_graphs=not a.eager)
    host = tr._stage_inputs(tokens)
    dev = {k: v.cuda() for k, v in host.items()}
    from paper_2502_19913_b200 import native
    for i in range(a.steps):
        if a.gemm_log and a.eager:
            native.record_gemms(True)
            native.take_gemm_log()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = tr.step(dev)
        torch.cuda.synchronize()
        print(f"step {i}: loss {r['loss']:.4f} {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    if a.gemm_log and a.eager:
        import json
        with open(a.gemm_log, "w") as f:
            json.dump([list(k) if k[0] != "group" else ["group", [list(x) for x in k[1]], k[2], k[3]]
                       for k in native.take_gemm_log()], f)


if __name__ == "__main__":
    main()
