"""Per-launch cost of small tcgen05 GEMMs and a trivial kernel, replayed back to back in a CUDA graph
(fixed overhead = launch + prologue + pipeline fill + last epilogue + teardown).

    python tools/launch_overhead.py
"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2502_19913_b200 import native
dev = "cuda"
def t(M, N, K, reps=50):
    A = torch.randn(M, K, device=dev).bfloat16(); B = torch.randn(N, K, device=dev).bfloat16(); C = torch.empty(M, N, device=dev).bfloat16()
    f = lambda: native.gemm(A, B, C, M=M, N=N, K=K, lda=K, ldb=K, ldc=N)
    for _ in range(3): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): f()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    print(M, N, K, round(s.elapsed_time(e) / reps * 1e3, 2), "us per launch")
for shp in [(256, 256, 64), (256, 256, 1024), (4096, 256, 1024), (256, 4096, 1024), (4096, 1024, 1024), (4096, 3072, 1024)]:
    t(*shp)
x = torch.empty(1 << 20, device=dev)
def e():
    native.sum_f32(x, 16, x[:1])
for _ in range(3): e()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(50): e()
g.replay(); torch.cuda.synchronize()
s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s_.record(); g.replay(); e_.record(); torch.cuda.synchronize()
print("tiny sum kernel", round(s_.elapsed_time(e_) / 50 * 1e3, 2), "us per launch")
