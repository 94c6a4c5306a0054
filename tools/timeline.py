"""Planned vs executed timeline of one SkipPipe iteration.

    python tools/timeline.py [--config C2] [--out profiles/r01_timeline] [--warmup 3]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/timeline.py ...

Writes <out>_planned.{csv,svg} (the simulator's trace for the plan) and <out>_executed_g<N>.{csv,svg}
(CUDA-event times of every op on every rank, merged on rank 0; each rank's clock starts at its
own iteration-start event, after a barrier).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_19913_b200.configs import get_config  # noqa: E402
from paper_2502_19913_b200.executor import Trainer  # noqa: E402
from paper_2502_19913_b200.gantt import emit_gantt, trace_csv  # noqa: E402
from paper_2502_19913_b200.model import synthetic_tokens  # noqa: E402
from paper_2502_19913_b200.simulator import simulate  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--out", default="profiles/r01_timeline")
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rc = get_config(a.config)
    if rank == 0:
        plan = simulate(rc.schedule(), rc.topology(), rc.sim_config(record_trace=True))
        with open(a.out + "_planned.csv", "w") as f:
            f.write(trace_csv(plan.trace))
        with open(a.out + "_planned.svg", "w") as f:
            f.write(emit_gantt(plan, rc.topology().n, f"{a.config} planned (simulator, planning times): "
                                                       f"{plan.iteration_makespan:.1f} ms"))
    tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T)
    tr = Trainer(rc.schedule(), rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split,
                 rank=rank, world=world, device=local)
    host = tr._stage_inputs(tokens)
    for _ in range(a.warmup):
        tr.step(host)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    rep = tr.make_report(tr.step(host, timing=True))
    rows = rep.trace
    mk = rep.iteration_makespan
    if world > 1:
        gathered = [None] * world
        dist.gather_object((rows, mk), gathered if rank == 0 else None, dst=0)
        if rank == 0:
            rows = [r for g in gathered for r in g[0]]
            mk = max(g[1] for g in gathered)
    if rank == 0:
        rep.trace, rep.iteration_makespan = rows, mk
        tag = f"{a.out}_executed_g{world}"
        with open(tag + ".csv", "w") as f:
            f.write(trace_csv(rows))
        with open(tag + ".svg", "w") as f:
            f.write(emit_gantt(rep, rc.topology().n, f"{a.config} executed on {world} B200 (CUDA events, "
                                                      f"placement {tr.placement}): {mk:.1f} ms"))
        print(f"planned {plan.iteration_makespan:.2f} ms (planning units), executed {mk:.2f} ms on {world} GPU(s)")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
