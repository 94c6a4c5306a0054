"""Multi-process host logic on CPU (gloo, world_size 2, 4 and 8): every rank derives the same hop
plan from the same schedule and posts sends/receives in global op order, so each message lands on
the intended receive — the property the NCCL P2P hops of the multi-GPU executor rely on."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_19913_b200.configs import get_config
from paper_2502_19913_b200.executor import allreduce_points, balanced_placement, hop_plan, static_slots
from paper_2502_19913_b200.simulator import simulate


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rc = get_config(cfg_name)
        sch = rc.schedule()
        rep = simulate(sch, rc.topology(), rc.sim_config())
        ops = rep.ops
        paths = {a: sch.paths[a].nodes for a in sch.paths}
        placement = balanced_placement(rep, rc.topology().n, world)  # the Trainer's default
        plan = hop_plan(ops, paths, placement)
        got, sent, pending = [], 0, []
        for idx, (op, hop) in enumerate(zip(ops, plan)):
            if hop is None:
                continue
            nv, name, src_rank, dst_rank, consumer = hop
            assert src_rank == placement[op.node]
            if src_rank == dst_rank:
                continue
            if rank == src_rank:
                pending.append(dist.isend(torch.tensor([idx, op.mb, nv]), dst_rank))
                sent += 1
            elif rank == dst_rank:
                buf = torch.zeros(3, dtype=torch.int64)
                dist.recv(buf, src_rank)
                got.append((idx, tuple(buf.tolist()), (idx, op.mb, nv)))
        for w in pending:
            w.wait()
        dist.barrier()
        q.put((rank, sent, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [(2, "C2"), (4, "C2"), (8, "C2"), (2, "C1"), (8, "C2-rb"), (4, "C2-rb"),
                                       (4, "C2-m4"), (8, "C2-m4")])
def test_cross_rank_hops_match(world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total_sent = sum(r[1] for r in results)
    received = [g for r in results for g in r[2]]
    assert total_sent == len(received) > 0
    for idx, got, want in received:
        assert got == want, (idx, got, want)


def test_static_slots_respect_tc1():
    rc = get_config("C2")
    sch = rc.schedule()
    slot_of, n_slots = static_slots(sch, rc.topology().n)
    assert max(n_slots) <= rc.m                       # TC1 => at most m slots per node
    for (a, v), j in slot_of.items():
        assert 0 <= j < n_slots[v] and v in sch.paths[a].nodes


def test_rebalanced_split_config():
    """C2-rb: S0 gets 3 of the 24 layers (it also runs embedding, head and loss
    for every microbatch); at 8 GPUs (one logical node per GPU) the busiest node's simulated load
    drops below the equal split's, and the full-pipeline comparator uses the same split."""
    eq, rb = get_config("C2"), get_config("C2-rb")
    assert rb.layers == [3, 7, 7, 7] and sum(rb.layers) == rb.model.n_layers
    assert get_config("C2-rb-full").layers == [3, 7, 7, 7] and get_config("C2-rb-full").kind == "full"
    busy_eq = simulate(eq.schedule(), eq.topology(), eq.sim_config()).node_busy
    busy_rb = simulate(rb.schedule(), rb.topology(), rb.sim_config()).node_busy
    assert max(busy_rb) < max(busy_eq)
    placement = balanced_placement(simulate(rb.schedule(), rb.topology(), rb.sim_config()), rb.topology().n, 8)
    assert sorted(placement) == list(range(8))


def test_memory_capacity_variant():
    """C2-m4: m = 4 microbatches per node (TC1) -> 8 agents; paths still satisfy TC1 (<= 4 per
    node) and the plan's makespan drops against m = 2 (fewer bubbles per wave)."""
    from paper_2502_19913_b200.scheduler import node_path_counts

    m2, m4 = get_config("C2"), get_config("C2-m4")
    assert m4.m == 4 and len(m4.schedule().agents) == 8 and m4.layers == m2.layers
    assert max(node_path_counts(m4.schedule().paths, m4.topology().n)) <= 4
    ms2 = simulate(m2.schedule(), m2.topology(), m2.sim_config()).iteration_makespan
    ms4 = simulate(m4.schedule(), m4.topology(), m4.sim_config()).iteration_makespan
    assert ms4 < ms2
    assert get_config("C2-rb-m4").layers == [3, 7, 7, 7] and get_config("C2-rb-m4-full").kind == "full"


@pytest.mark.parametrize("cfg,world", [("C2", 2), ("C2-m4", 2), ("C2-m4", 4), ("C2-rb", 8)])
def test_allreduce_order_is_global(cfg, world):
    """Replica all-reduces are placed at each stage's last op in the global op order: the same
    positions on every rank (independent of which stages a rank holds), every hosting rank has
    all its ops of the stage before that point, and stages come out in one order."""
    rc = get_config(cfg)
    rep = simulate(rc.schedule(), rc.topology(), rc.sim_config())
    node_stage = rc.assignment.node_stage()
    placement = balanced_placement(rep, rc.topology().n, world)
    cross = [st for st in range(rc.s) if len({placement[v] for v in range(rc.topology().n) if node_stage[v] == st}) > 1]
    pts = allreduce_points(rep.ops, node_stage, cross)
    order = [st for i in sorted(pts) for st in pts[i]]
    assert sorted(order) == sorted(cross)
    for r in range(world):
        mine = [st for st in cross if any(placement[v] == r for v in range(rc.topology().n) if node_stage[v] == st)]
        assert allreduce_points(rep.ops, node_stage, mine) == {i: [s for s in v if s in mine] for i, v in pts.items()
                                                               if any(s in mine for s in v)}
        for i, sts in pts.items():
            for st in sts:
                assert all(j <= i for j, op in enumerate(rep.ops) if node_stage[op.node] == st and placement[op.node] == r)
