"""Graph-replayed timing of one C2 decoder layer's grouped weight-gradient launch (the four
dW = dY^T X problems of executor.StageProgram.layer_bwd in one spx_gemm_f32_group launch),
with the GEMM pipeline probes selectable by SPX_GEMM_PROBE (benchmarking only).

    python tools/wgrad_bench.py [--config C2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19913_b200 import native  # noqa: E402
from paper_2502_19913_b200.configs import get_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    a = ap.parse_args()
    rc = get_config(a.config)
    c, n = rc.model, rc.b * rc.T
    d, f, qd, od = c.d, c.ffn, c.qkv_dim, c.n_heads * c.head_dim
    dev = "cuda"
    bf = dict(dtype=torch.bfloat16, device=dev)
    dgu, xn2, dqkv, xn1 = (torch.randn(n, 2 * f, **bf), torch.randn(n, d, **bf), torch.randn(n, qd, **bf),
                           torch.randn(n, d, **bf))
    dy, h, dxm, o = torch.randn(n, d, **bf), torch.randn(n, f, **bf), torch.randn(n, d, **bf), torch.randn(n, od, **bf)
    g_gu, g_qkv = torch.zeros(2 * f, d, device=dev), torch.zeros(qd, d, device=dev)
    g_down, g_o = torch.zeros(d, f, device=dev), torch.zeros(d, od, device=dev)
    group = [
        dict(A=dgu, B=xn2, C=g_gu, M=2 * f, N=d, K=n, lda=2 * f, ldb=d, ldc=d, beta=1.0),
        dict(A=dqkv, B=xn1, C=g_qkv, M=qd, N=d, K=n, lda=qd, ldb=d, ldc=d, beta=1.0),
        dict(A=dy, B=h, C=g_down, M=d, N=f, K=n, lda=d, ldb=f, ldc=f, beta=1.0),
        dict(A=dxm, B=o, C=g_o, M=d, N=od, K=n, lda=d, ldb=od, ldc=od, beta=1.0),
    ]
    native.gemm_set_workspace(None)
    fl = sum(2.0 * p["M"] * p["N"] * p["K"] for p in group)
    for _ in range(3):
        native.gemm_f32_group(group)
    torch.cuda.synchronize()
    iters = 20
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            native.gemm_f32_group(group)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / iters * 1e3
    print(f"{{\"config\": \"{a.config}\", \"probe\": \"{os.environ.get('SPX_GEMM_PROBE', '0')}\", \"us\": {us:.2f}, "
          f"\"tflops\": {fl / us / 1e6:.1f}}}", flush=True)


if __name__ == "__main__":
    main()
