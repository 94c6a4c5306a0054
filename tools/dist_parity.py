"""Multi-GPU parity driver (launched by tests/test_dist_gpu.py under torchrun):
config SPX_CONFIG (default C1; SPX_M overrides the microbatch count) on WORLD_SIZE GPUs vs the
fp32 oracle (run by every rank on its own GPU with TF32 off, as a checker) and vs the per-node op order
of the simulator.  Rank 0 prints one JSON line with the comparison results, including a SHA-256
of every stage's fp32 master weights after two steps (hops are pure copies, so every hop
transport must give the same bits)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import train_ref  # noqa: E402
from paper_2502_19913_b200.configs import get_config  # noqa: E402
from paper_2502_19913_b200.executor import Trainer  # noqa: E402
from paper_2502_19913_b200.model import init_params, synthetic_tokens  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    over = {"M": int(os.environ["SPX_M"])} if os.environ.get("SPX_M") else {}
    rc = get_config(os.environ.get("SPX_CONFIG", "C1"), **over)
    oracle_dev = f"cuda:{local}"
    torch.backends.cuda.matmul.allow_tf32 = False
    sch = rc.schedule()
    params = init_params(rc.model, rc.layers, seed=0)
    tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T, seed=1234)
    tr = Trainer(sch, rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split, params=params,
                 rank=rank, world=world, device=local, keep_grads=True)
    res = tr.step(tokens, timing=True)
    rep = tr.make_report(res)
    grads = tr.grads()
    gnorm = tr.grad_norm()
    res2 = tr.step(tokens)
    p2 = tr.params()
    digest = {st: hashlib.sha256(b"".join(p2[st][k].numpy().tobytes() for k in sorted(p2[st]))).hexdigest()
              for st in p2}
    # per-node order of the ops this rank executed vs the simulator's
    sim = {}
    for op in tr.ops:
        if tr.placement[op.node] == rank:
            sim.setdefault(op.node, []).append((op.kind, op.agent, op.wave))
    order_ok = rep.node_order == sim
    # every rank runs the fp32 oracle (on its own GPU, TF32 off) and compares the stages it hosts
    agents = sorted(a.id for a in sch.agents)
    mbs = train_ref.mb_stage_sequences({a: sch.paths[a].stages for a in agents}, agents, rc.M)
    ref = train_ref.iteration(rc.model, rc.layers, params, mbs, tokens, update=False, device=oracle_dev)
    stage_cos = {}
    for st, g in grads.items():
        a = torch.cat([g[k].reshape(-1) for k in sorted(g)]).double()
        b = torch.cat([ref["grads"][st][k].reshape(-1).cpu() for k in sorted(g)]).double()
        stage_cos[f"{rank}:{st}"] = [torch.nn.functional.cosine_similarity(a, b, dim=0).item(),
                                     ((a - b).norm() / b.norm()).item()]
    out = [None] * world
    dist.all_gather_object(out, {"rank": rank, "stage_cos": stage_cos, "order_ok": order_ok, "digest": digest})
    if rank == 0:
        params_sha, cos_all = {}, {}
        for o in out:
            cos_all.update(o["stage_cos"])
            for st, h in o["digest"].items():
                assert params_sha.setdefault(st, h) == h, f"stage {st} replicas differ after the update"
        print(json.dumps({"world": world, "config": rc.name, "M": rc.M, "hop": tr.hop_transport,
                          "engine": tr.hop_engine, "params_sha": {str(k): v for k, v in sorted(params_sha.items())},
                          "loss": res["loss"], "loss2": res2["loss"], "ref_loss": ref["loss"],
                          "order_ok": all(o["order_ok"] for o in out), "stage_cos_rel": cos_all,
                          "grad_norm": gnorm, "ref_grad_norm": ref["grad_norm"]}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
