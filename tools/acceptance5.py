"""SPEC.md:536 acceptance 5 (throughput ordering) at the spec's scale: 50 sampled topologies per
§4.1 profile (20 nodes / s=6 / k=33 %, 18 nodes / s=4 / k=25 %).  Per topology: SkipPipe,
SkipPipe without TC2, DT-FM-skip and compensated DT-FM full (the largest node count divisible by
s, credited by compensate()), simulated over M = 2 * lcm(|agents|) microbatches.  Sampled
topologies on which phase 1 finds no CC3-feasible candidate (InfeasibleError) are replaced by the
next seed and listed.

Usage: python tools/acceptance5.py --profile 18|20 [--seeds 50] [--out FILE.jsonl]
Prints one JSON line per topology and a summary line (means, speedups, ordering counts).
"""

import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_19913_b200 import scheduler as S  # noqa: E402
from paper_2502_19913_b200.allocation import GAConfig, allocate  # noqa: E402
from paper_2502_19913_b200.baselines import compensate, dtfm_full, dtfm_skip, skippipe_no_tc2  # noqa: E402
from paper_2502_19913_b200.errors import InfeasibleError  # noqa: E402
from paper_2502_19913_b200.scheduler import make_agents  # noqa: E402
from paper_2502_19913_b200.simulator import SimConfig, simulate  # noqa: E402
from paper_2502_19913_b200.topology import TopologyProfile, sample_topology  # noqa: E402

PROFILES = {"18": (3, 6, 4, 25.0), "20": (4, 5, 6, 100 / 3)}
MSG = 4 * 1024 * 2048 * 2.0  # activation bytes of one microbatch (b=4, T=1024, d=2048, bf16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--profile", choices=sorted(PROFILES), required=True)
    ap.add_argument("--seeds", type=int, default=50)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    regions, per, s, k = PROFILES[a.profile]
    out = open(a.out, "w") if a.out else None
    rows, infeasible = [], []
    t_all = time.time()
    seed = -1
    while len(rows) < a.seeds:  # topologies on which phase 1 finds no CC3-feasible candidate are replaced
        seed += 1
        t0 = time.time()
        T = sample_topology(TopologyProfile(regions=regions, nodes_per_region=per, seed=seed))
        A = allocate(T, s, k, MSG, GAConfig(population=32, generations=40, seed=seed))
        # M = 2 * lcm(|agents| of SkipPipe, |agents| of DT-FM full): the iteration every arm is
        # simulated over, also what the scheduler's final selection simulates (sim_microbatches)
        n_full = T.n - T.n % s
        n_sp = len(make_agents(A, T.mem_capacity))
        n_fa = (n_full // s) * T.mem_capacity
        M = 2 * (n_sp * n_fa // math.gcd(n_sp, n_fa))
        cfg = S.SchedulerConfig(k=k, msg_bytes=MSG, sim_microbatches=M)
        try:
            sp, nt, ds = S.schedule(T, A, cfg), skippipe_no_tc2(T, A, cfg), dtfm_skip(T, A, cfg)
        except InfeasibleError:
            infeasible.append(seed)
            continue
        T_full = T.restrict(list(range(n_full)))
        full = dtfm_full(T_full, s, msg_bytes=MSG)
        assert (len(sp.agents), len(full.agents)) == (n_sp, n_fa)
        sc = SimConfig(total_microbatches=M, msg_bytes=MSG)
        r = {"profile": a.profile, "seed": seed, "M": M,
             "skippipe": simulate(sp, T, sc).iteration_makespan,
             "no_tc2": simulate(nt, T, sc).iteration_makespan,
             "dtfm_skip": simulate(ds, T, sc).iteration_makespan,
             "dtfm_full_comp": compensate(simulate(full, T_full, sc).iteration_makespan, n_full, T.n),
             "resolved": sp.resolved, "resolved_no_tc2": nt.resolved, "s": round(time.time() - t0, 1)}
        rows.append(r)
        line = json.dumps(r)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
            out.flush()
    mean = lambda key: sum(r[key] for r in rows) / len(rows)  # noqa: E731
    summ = {"profile": a.profile, "topologies": len(rows),
            "mean_ms": {key: round(mean(key), 1) for key in ("skippipe", "no_tc2", "dtfm_skip", "dtfm_full_comp")},
            "speedup_vs_dtfm_full": round(mean("dtfm_full_comp") / mean("skippipe") - 1, 4),
            "speedup_vs_no_tc2": round(mean("no_tc2") / mean("skippipe") - 1, 4),
            "runs_skippipe_le_no_tc2": sum(r["skippipe"] <= r["no_tc2"] + 1e-9 for r in rows),
            "runs_no_tc2_le_dtfm_skip": sum(r["no_tc2"] <= r["dtfm_skip"] + 1e-9 for r in rows),
            "runs_skippipe_lt_dtfm_skip": sum(r["skippipe"] < r["dtfm_skip"] for r in rows),
            "resolved": sum(r["resolved"] for r in rows), "infeasible_seeds": infeasible,
            "minutes": round((time.time() - t_all) / 60, 1)}
    print(json.dumps({"summary": summ}), flush=True)
    if out:
        out.write(json.dumps({"summary": summ}) + "\n")


if __name__ == "__main__":
    main()
