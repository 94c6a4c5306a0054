"""Benchmark: SkipPipe partial-pipeline training iteration on B200 (BASELINE.json metric:
"iteration time (ms) & tokens/s, LLaMa-500M 25% skip, 1/2/4/8 B200 vs full PP").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One "step" = one synchronous training iteration of config C2 (LLaMa-500M, 4 stages x 2
replicas, 25% skip, M=32 microbatches of 4x1024 tokens = 131,072 tokens) — F, loss and B of
every microbatch along its scheduled path, replica gradient sync, clip and AdamW.  Inputs are
synthetic uniform token ids; weights random N(0, 0.02).  At N=1 all 8 logical nodes are
resident on one GPU; at N>1 (torchrun, one process per GPU) the nodes are placed over the
GPUs and hops go over NVLink (see executor.py; `hops` in the JSON line reports their bandwidth).

`value` is tokens/s with the step's inputs already in HBM; `e2e` is the same metric through the
public ``Trainer.step(tokens)`` call with host token buffers (H2D staging and the loss readback
inside the timed region).  `--impl reference` times the CPU fp32 oracle (the reference ships no
executor) on a bounded sample of the same workload on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # per-node compute streams (executor.py)
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "iteration time (ms) & tokens/s, LLaMa-500M 25% skip, 1/2/4/8 B200 vs full PP"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int = 0):
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                for nm, val in zip(names, f[5:9]):
                    if val.lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(rc, budget_s: float = 20.0) -> dict:
    """CPU fp32 oracle on a bounded sample: one microbatch path (F through its stages, loss, B)
    of the same model, b=1, timed on all host threads; reported as tokens/s."""
    import torch

    from oracle import train_ref
    from paper_2502_19913_b200.model import init_params, synthetic_tokens

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    params = init_params(rc.model, rc.layers, seed=0)
    sch = rc.schedule()
    agents = sorted(a.id for a in sch.agents)
    stages = sch.paths[agents[0]].stages
    tokens = synthetic_tokens(rc.model, 1, 1, rc.T, seed=1234)
    times = []
    t_end = time.time() + budget_s
    while time.time() < t_end or not times:
        t0 = time.perf_counter()
        train_ref.iteration(rc.model, rc.layers, params, [stages], tokens, update=False)
        times.append(time.perf_counter() - t0)
        if len(times) >= 3:
            break
    sec = statistics.median(times)
    return {"value": rc.T / sec, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"1 microbatch (1x{rc.T} tokens) along path stages {list(stages)}: F+loss+B, fp32 torch CPU, "
                      f"median of {len(times)}"}


def c1_iteration() -> dict:
    """A directly timed full training iteration of config C1 (BASELINE configs[0], the tiny
    CPU-runnable case: M=8 microbatches of 2x256 tokens along the scheduled paths, loss, backward,
    clip and AdamW) on the CPU fp32 oracle, all host threads -- no extrapolation."""
    import torch

    from oracle import train_ref
    from paper_2502_19913_b200.configs import get_config
    from paper_2502_19913_b200.model import init_params, synthetic_tokens

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    rc = get_config("C1")
    sch = rc.schedule()
    agents = sorted(a.id for a in sch.agents)
    mbs = train_ref.mb_stage_sequences({a: sch.paths[a].stages for a in agents}, agents, rc.M)
    params = init_params(rc.model, rc.layers, seed=0)
    tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T, seed=1234)
    t0 = time.perf_counter()
    out = train_ref.iteration(rc.model, rc.layers, params, mbs, tokens, update=True)
    sec = time.perf_counter() - t0
    return {"config": "C1", "ms": sec * 1e3, "tokens_per_s": rc.M * rc.tokens_per_mb / sec, "cores": threads,
            "loss": out["loss"]}


def run_reference(args, rc):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t0 = time.time()
    cb = cpu_baseline(rc, budget_s=min(30.0, 10.0 * max(1, args.steps)))
    c1 = c1_iteration()
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": rc.M * rc.tokens_per_mb / cb["value"] * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": rc.name, "model": rc.model.name, "global_batch": rc.M * rc.b, "seq_len": rc.T,
                       "parallelism": "cpu"},
            "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0},
            "c1_iteration": c1, "wall_s": time.time() - t0}
    print(json.dumps(line), flush=True)


def gemm_roofline(tr, peak_tflops: float, reps: int = 10) -> dict:
    """Per-launch timing of every tcgen05 GEMM of one iteration (same shapes, layouts, epilogues
    and buffers as inside the captured graphs): ``reps`` back-to-back launches captured in a CUDA
    graph and replayed on the executor's stream, timed with CUDA events."""
    import torch

    from paper_2502_19913_b200 import native

    calls = native.recorded_gemms()
    counts = tr.gemm_counts_per_step()
    # DRAM bytes per launch of each shape from the committed ncu capture (profiles/), if present
    traffic_by_shape = {}
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_gemm_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic_by_shape = {k: v["dram_bytes_per_launch"] for k, v in json.load(f)["per_shape"].items()}
    t_bytes, t_count = 0.0, 0
    s = tr.stream
    total_flops, total_ms = 0.0, 0.0
    per = {}
    for key, (_, fn) in calls.items():
        count = counts.get(key, 0)
        # the same launches replayed from a CUDA graph (as in the iteration): device time per
        # launch without host launch gaps
        with torch.cuda.stream(s):
            fn()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        with torch.cuda.stream(s):
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        if key[0] == "group":  # grouped wgrad launch: ("group", ((M, N, K), ...), a_mn, b_mn)
            fl = sum(2.0 * m * n * k for (m, n, k) in key[1])
        else:
            fl = 2.0 * key[0] * key[1] * key[2]
        total_flops += fl * count
        total_ms += ms * count
        per[str(key)] = {"launches_per_step": count, "us": round(ms * 1e3, 2), "tflops": round(fl / ms / 1e9, 1)}
        if str(key) in traffic_by_shape:
            per[str(key)]["dram_bytes"] = traffic_by_shape[str(key)]
            t_bytes += traffic_by_shape[str(key)] * count
            t_count += count
    ach = total_flops / total_ms / 1e9 if total_ms else 0.0
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": round(ach / peak_tflops, 4),
            "traffic": round(t_bytes / t_count) if t_count else None,
            "traffic_note": "dram read+write bytes per GEMM launch, launch-weighted over the iteration's shapes "
                            "(ncu capture profiles/r02_gemm_traffic.json; per shape in per_shape)",
            "kernel": "spx gemm_bf16_kernel (tcgen05, all shapes)",
            "gemm_ms_per_step": round(total_ms, 3), "per_shape": per}


NVLINK_GBS = 900.0  # NVLink 5 per GPU per direction (18 links x 50 GB/s), nominal: no measured peak


def hop_bandwidth(tr, ms_step: float, reps: int = 20) -> dict:
    """Path-hop transport (north_star: "for the P2P hops as a fraction of NVLink bandwidth").

    Counts the iteration's cross-GPU hops from the executor's hop plan (every rank derives the
    same plan), then times one hop message (an [n, d] bf16 activation or activation gradient)
    sent rank 0 -> rank 1 with the executor's own transport (a spx_hop_push into a rank-1 slot,
    or NCCL send/recv on the pair communicator), alone on a side stream, ``reps`` back-to-back
    messages bracketed by CUDA events on that stream.
    All ranks must call it (collective barrier); only ranks 0 and 1 move data."""
    import torch
    import torch.distributed as dist

    from paper_2502_19913_b200 import native

    cross = sum(1 for h in tr.hops if h is not None and h[2] != h[3])
    c = tr.cfg
    n = tr.b * tr.T
    msg = n * c.d * 2
    out = {"cross_gpu_hops_per_step": cross, "msg_bytes": msg, "bytes_per_step": cross * msg,
           "demand_gbs": round(cross * msg / (ms_step / 1e3) / 1e9, 2)}
    buf = torch.empty(n, c.d, dtype=torch.bfloat16, device=tr.dev)
    s = torch.cuda.Stream(tr.dev)
    peer = tr.hop_transport == "peer"
    dist.barrier()
    torch.cuda.synchronize(tr.dev)
    t = torch.zeros(1, device=tr.dev)
    if tr.rank in (0, 1):
        other = 1 - tr.rank
        if peer:   # a hop-receive slot hosted on rank 1 (same choice on both ranks)
            key = min(k for k in (tr._peer_addr if tr.rank == 0 else tr._flag_expect) if tr.placement[k[0]] == 1)
        for it in range(2):                        # warm-up pass, then the timed pass
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                if peer and tr.rank == 0:
                    tr._push(tr._peer_addr[key], buf, tr._peer_flag[key], s)
                elif peer:
                    tr._flag_expect[key] += tr.hop_inc
                    native.hop_wait(tr._flag_local[key], tr._flag_expect[key], stream=s)
                else:
                    with torch.cuda.stream(s):
                        if tr.rank == 0:
                            dist.send(buf, other, group=tr._pair[other])
                        else:
                            dist.recv(buf, other, group=tr._pair[other])
            e1.record(s)
            torch.cuda.synchronize(tr.dev)
        if tr.rank == 0:
            t[0] = e0.elapsed_time(e1) * 1e3 / reps
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    us = float(t.item())
    gbs = msg / (us / 1e6) / 1e9
    out.update({"hop_us": round(us, 2), "achieved_gbs": round(gbs, 1), "peak_gbs": NVLINK_GBS,
                "peak_kind": "nominal NVLink 5 per direction", "frac": round(gbs / NVLINK_GBS, 4),
                "hop_ms_per_step_if_serial": round(cross * us / 1e3, 3),
                "transport": tr.hop_transport + (f"/{tr.hop_engine}" if peer else ""),
                "ctas": tr.hop_ctas if peer and tr.hop_engine == "sm" else None,
                "how": (f"rank0->rank1 {'spx_hop_push_ce' if tr.hop_engine == 'ce' else 'spx_hop_push'} into a "
                        "rank-1 slot over NVLink peer memory + arrival flag, rank 1 waiting on it" if peer
                        else "rank0->rank1 NCCL send/recv on the executor's pair group") +
                       f", CUDA events, {reps} back-to-back messages after a warm-up pass"})
    return out


def time_full_pp(args, rc_name, rank=0, world=1, local=0, variant="-full", over=None):
    """Same protocol on the full sequential pipeline (dtfm_full, k=0) of the same model on the same
    GPUs — the metric's "vs full PP" comparison — or on another executable baseline variant
    ("-dtfmskip", "-notc2"; configs.VARIANTS).  Returns ms/step (max over ranks)."""
    import torch

    from paper_2502_19913_b200.configs import get_config
    from paper_2502_19913_b200.executor import Trainer
    from paper_2502_19913_b200.model import synthetic_tokens

    rf = get_config(rc_name + variant, **(over or {}))
    tokens = synthetic_tokens(rf.model, rf.M, rf.b, rf.T, seed=1234)
    tr = Trainer(rf.schedule(), rf.topology(), rf.sim_config(), rf.model, rf.assignment, b=rf.b, T=rf.T, split=rf.split,
                 rank=rank, world=world, device=local)
    dev_inputs = {k: v.cuda() for k, v in tr._stage_inputs(tokens).items()}
    for _ in range(max(1, args.warmup)):
        tr.step(dev_inputs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    e0.record(tr.stream)
    for _ in range(args.steps):
        tr.step(dev_inputs)
    e1.record(tr.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device=tr.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    del tr
    torch.cuda.empty_cache()
    return ms, rf


def time_baselines(args, rc_name, ms, tok, rank=0, world=1, local=0):
    """Executed DT-FM-skip and SkipPipe-without-TC2 schedules next to SkipPipe."""
    out = {}
    for variant, label in (("-dtfmskip", "dtfm_skip"), ("-notc2", "skippipe_no_tc2")):
        bms, rb = time_full_pp(args, rc_name, rank=rank, world=world, local=local, variant=variant)
        out[label] = {"workload": rb.name, "ms_per_step": round(bms, 3), "tokens_per_s": round(tok / (bms / 1e3), 1),
                      "skippipe_speedup": round(bms / ms, 4)}
    return out


def time_variants(args, rc, ms, tok, rank=0, world=1, local=0):
    """Opt-in B200 settings of the headline config measured beside it, same protocol, same GPUs:
    C2-m4 (memory capacity m = 4: 8 agents in flight).  Skipped with --no-variants
    and for other configs."""
    if args.no_variants or rc.name != "C2":
        return None
    out = {}
    for variant, label in (("-m4", "C2-m4 (m=4)"),):
        vms, rv = time_full_pp(args, rc.name, rank=rank, world=world, local=local, variant=variant)
        out[rv.name] = {"what": label, "ms_per_step": round(vms, 3), "tokens_per_s": round(tok / (vms / 1e3), 1),
                        "vs_headline": round(ms / vms, 4)}
    return out


def time_sweep(args, ms_c2, tok, rank=0, world=1, local=0):
    """BASELINE.json configs[4]: LLaMa-500M skip-ratio sweep 0/25/50 % against the full sequential
    pipeline, same GPUs, same protocol.  0 % is SkipPipe's scheduler with k=0 (paths may still
    cross replicas); "full" is DT-FM's disjoint sequential pipelines.  25 % is the headline run."""
    full_ms, _ = time_full_pp(args, "C2", rank=rank, world=world, local=local, variant="-full")
    pts = []
    for pct, name, over in ((0, "C2", {"k": 0}), (25, None, None), (50, "C5", None)):
        ms = ms_c2 if name is None else time_full_pp(args, name, rank=rank, world=world, local=local, variant="",
                                                     over=over)[0]
        pts.append({"skip_pct": pct, "ms_per_step": round(ms, 3), "tokens_per_s": round(tok / (ms / 1e3), 1),
                    "vs_full_pp_speedup": round(full_ms / ms, 4)})
    return {"full_pp_ms_per_step": round(full_ms, 3), "points": pts}


def run_ours(args, rc):
    import torch

    from paper_2502_19913_b200 import native
    from paper_2502_19913_b200.executor import Trainer
    from paper_2502_19913_b200.model import synthetic_tokens

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        return run_ours_dist(args, rc)
    torch.cuda.set_device(0)
    burst, sustained, hbm, peak_kind = _peaks()
    tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T, seed=1234)
    native.record_gemms(True)
    tr = Trainer(rc.schedule(), rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split)
    native.record_gemms(False)
    launches = tr.launches_per_step()
    host = tr._stage_inputs(tokens)
    dev_inputs = {k: v.cuda() for k, v in host.items()}
    # L2 (126 MB) is far smaller than one step's working set (~tens of GB of activations and
    # weights), so no explicit flush is needed between steps.
    for _ in range(args.warmup):
        tr.step(dev_inputs)
    torch.cuda.synchronize()
    s = tr.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(args.steps):
            res = tr.step(dev_inputs)
        e1.record(s)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    tok = rc.M * rc.tokens_per_mb
    value = tok / (ms / 1e3)
    # e2e through the public API: host token tensor in, host loss out, every step
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = tr.step(tokens)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    flops = rc.train_flops()
    roof = gemm_roofline(tr, burst)
    h2d = tr.h2d_bytes(tokens)
    cb = cpu_baseline(rc, budget_s=15.0) if not args.no_cpu_baseline else None
    full = None
    if not args.no_full_pp and rc.kind == "skippipe":
        del tr
        torch.cuda.empty_cache()
        fms, rf = time_full_pp(args, rc.name)
        full = {"workload": rf.name, "kind": "dtfm_full (k=0, disjoint sequential pipelines)",
                "ms_per_step": round(fms, 3), "tokens_per_s": round(tok / (fms / 1e3), 1),
                "skippipe_speedup": round(fms / ms, 4)}
    bl = time_baselines(args, rc.name, ms, tok) if args.baselines and rc.kind == "skippipe" else None
    sw = time_sweep(args, ms, tok) if args.sweep and rc.name == "C2" else None
    var = time_variants(args, rc, ms, tok)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": rc.name, "model": rc.model.name, "global_batch": rc.M * rc.b, "seq_len": rc.T,
                   "microbatches": rc.M, "tokens_per_step": tok, "stages": rc.s, "replicas": rc.sizes,
                   "skip_pct": rc.k, "m": rc.m, "layer_split": rc.layers,
                   "swapped_paths": rc.swapped_paths(), "parallelism": f"pp-skip({rc.s}x{rc.sizes[0]} logical nodes on 1 GPU)",
                   "l2_flush": "inputs+activations per step >> 126 MB L2", "kind": rc.kind},
        "loss": round(res["loss"], 5),
        "e2e": {"value": round(tok / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4 * rc.M},
        "gpu_launches": launches,
        "step_tflops": round(flops / (ms / 1e3) / 1e12, 1),
        "step_tensor_frac": round(flops / (ms / 1e3) / 1e12 / sustained, 4),
        "roofline": {**roof, "peak_kind": f"{peak_kind} burst bf16 (GEMMs timed alone)"},
        "cpu_baseline": cb,
        "vs_full_pp": full,
        "baselines": bl,
        "skip_sweep": sw,
        "variants": var,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def run_ours_dist(args, rc):
    """N>1: torchrun, one process per GPU.  Logical nodes are placed rank = node mod N; hops
    between ranks are NCCL P2P over NVLink, replicated stages are all-reduced per stage group.
    Total work per step is the fixed C2 iteration (strong scaling); time = max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2502_19913_b200 import native
    from paper_2502_19913_b200.executor import Trainer
    from paper_2502_19913_b200.model import synthetic_tokens

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch with torchrun --nproc-per-node {args.gpus}")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    burst, sustained, hbm, peak_kind = _peaks()
    tokens = synthetic_tokens(rc.model, rc.M, rc.b, rc.T, seed=1234)
    native.record_gemms(True)
    tr = Trainer(rc.schedule(), rc.topology(), rc.sim_config(), rc.model, rc.assignment, b=rc.b, T=rc.T, split=rc.split,
                 rank=rank, world=world, device=local)
    native.record_gemms(False)
    launches = torch.tensor([tr.launches_per_step()], device=tr.dev)
    placement = list(tr.placement)
    dist.all_reduce(launches)
    host = tr._stage_inputs(tokens)
    dev_inputs = {k: v.cuda() for k, v in host.items()}
    for _ in range(args.warmup):
        tr.step(dev_inputs)
    torch.cuda.synchronize()
    s = tr.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(args.steps):
            res = tr.step(dev_inputs)
        e1.record(s)
        torch.cuda.synchronize()
        dist.barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms_local], device=tr.dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    tok = rc.M * rc.tokens_per_mb
    # e2e through the public API with host tokens
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tr.step(tokens)
    torch.cuda.synchronize()
    e2e_local = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([e2e_local, float(tr.h2d_bytes(tokens))], device=tr.dev)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm)
    flops = rc.train_flops()
    roof = gemm_roofline(tr, burst) if rank == 0 else None
    hops = hop_bandwidth(tr, ms)
    full = None
    if not args.no_full_pp and rc.kind == "skippipe":
        del tr
        torch.cuda.empty_cache()
        fms, rf = time_full_pp(args, rc.name, rank=rank, world=world, local=local)
        full = {"workload": rf.name, "kind": "dtfm_full (k=0, disjoint sequential pipelines)",
                "ms_per_step": round(fms, 3), "tokens_per_s": round(tok / (fms / 1e3), 1),
                "skippipe_speedup": round(fms / ms, 4)}
    sw = time_sweep(args, ms, tok, rank, world, local) if args.sweep and rc.name == "C2" else None
    bl = time_baselines(args, rc.name, ms, tok, rank, world, local) if args.baselines and rc.kind == "skippipe" \
        else None
    var = time_variants(args, rc, ms, tok, rank, world, local)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(tok / (ms / 1e3), 1), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": rc.name, "model": rc.model.name, "global_batch": rc.M * rc.b, "seq_len": rc.T,
                       "microbatches": rc.M, "tokens_per_step": tok, "stages": rc.s, "replicas": rc.sizes,
                       "skip_pct": rc.k, "m": rc.m, "layer_split": rc.layers,
                   "swapped_paths": rc.swapped_paths(), "placement": placement,
                       "parallelism": f"pp-skip({rc.s}x{rc.sizes[0]} logical nodes over {world} GPUs)+dp-allreduce",
                       "l2_flush": "inputs+activations per step >> 126 MB L2", "kind": rc.kind},
            "loss": round(res["loss"], 5),
            "e2e": {"value": round(tok / (float(mx[0].item()) / 1e3), 1), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(sm[1].item()), "d2h_bytes_per_step": 4 * rc.M},
            "gpu_launches": int(launches.item()),
            "step_tflops": round(flops / (ms / 1e3) / 1e12, 1),
            "step_tensor_frac": round(flops / (ms / 1e3) / 1e12 / (sustained * world), 4),
            "roofline": {**roof, "peak_kind": f"{peak_kind} burst bf16 (GEMMs timed alone, rank 0)"},
            "hops": hops,
            "vs_full_pp": full,
            "baselines": bl,
            "skip_sweep": sw,
            "variants": var,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-pp", action="store_true", help="skip the full sequential pipeline comparison")
    ap.add_argument("--no-variants", action="store_true", help="skip the C2-m4 variant measured beside the headline")
    ap.add_argument("--sweep", action="store_true",
                    help="also run the C5 skip-ratio sweep (0/25/50%% vs full PP) on the same GPUs")
    ap.add_argument("--baselines", action="store_true",
                    help="also execute the DT-FM-skip and SkipPipe-without-TC2 schedules (same protocol)")
    args = ap.parse_args()
    from paper_2502_19913_b200.configs import get_config

    rc = get_config(args.config)
    if args.impl == "reference":
        run_reference(args, rc)
    else:
        run_ours(args, rc)


if __name__ == "__main__":
    main()
