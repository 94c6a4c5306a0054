"""Bandwidth of the per-iteration update kernels (AdamW, replica-grad merge, grad-norm, grad zeroing).

    python tools/opt_bench.py [--n 46000000]

Each kernel is replayed from a CUDA graph (20 launches) and timed with CUDA events; the buffers
(n fp32 elements each, default ≈ one C2 stage) exceed L2, so every launch streams from HBM.
Algorithmic bytes: AdamW reads p, g, m, v (16 B) and writes p, m, v, bf16 p (14 B) per element;
add reads 2 and writes 1 fp32; sumsq reads 1; zero writes 1.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_19913_b200 import native  # noqa: E402


def timed(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=46_000_000)
    a = ap.parse_args()
    n, dev = a.n, "cuda:0"
    off = 1  # misaligned views select the scalar AdamW kernel
    buf = {k: torch.rand(n + off, device=dev) for k in ("p", "g", "m", "v")}
    pb = torch.empty(n + off, dtype=torch.bfloat16, device=dev)
    sc = torch.ones(1, device=dev)
    ws = torch.empty(native.sumsq_ws_floats(), device=dev)
    out = torch.empty(1, device=dev)
    rows = {}

    def adamw(o):
        return lambda: native.adamw(buf["p"][o:], buf["g"][o:], buf["m"][o:], buf["v"][o:], pb[o:], n=n, n_decay=n // 2,
                                    lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1, step=3,
                                    grad_scale=sc, stream=torch.cuda.current_stream())

    s = torch.cuda.current_stream
    rows["adamw_vec"] = (timed(adamw(0)), 30 * n)
    rows["adamw_scalar"] = (timed(adamw(1)), 30 * n)
    rows["add_f32"] = (timed(lambda: native.add_f32(buf["p"], buf["g"], n, stream=s())), 12 * n)
    rows["sumsq"] = (timed(lambda: native.sumsq(buf["g"], n, ws, out, stream=s())), 4 * n)
    rows["torch_zero"] = (timed(lambda: buf["m"].zero_()), 4 * (n + off))
    rows["torch_copy"] = (timed(lambda: buf["m"].copy_(buf["v"])), 8 * (n + off))
    res = {k: {"us": round(t, 1), "GB/s": round(b / t / 1e3, 1)} for k, (t, b) in rows.items()}
    print(json.dumps({"n": n, "kernels": res}))


if __name__ == "__main__":
    main()
