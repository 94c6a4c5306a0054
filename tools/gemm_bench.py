"""Time spx_gemm_bf16 on the llama-500m (config C2) stage shapes; compare with torch.matmul (cuBLAS).

Usage: python tools/gemm_bench.py [--only SUBSTRING] [--no-cublas]   (prints one line per shape)
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_19913_b200 import native  # noqa: E402

SHAPES = [
    # name, M, N, K, a_mn, b_mn, epi
    ("qkv fwd", 4096, 3072, 1024, False, False, native.EPI_BF16),
    ("qkv fwd+rope", 4096, 3072, 1024, False, False, "rope"),
    ("o fwd+res", 4096, 1024, 1024, False, False, native.EPI_BF16_RESID),
    ("gate/up fwd swiglu", 4096, 5632, 1024, False, False, native.EPI_SWIGLU),
    ("down fwd+res", 4096, 1024, 2816, False, False, native.EPI_BF16_RESID),
    ("head fwd", 4096, 32000, 1024, False, False, native.EPI_BF16),
    ("qkv dgrad", 4096, 1024, 3072, False, True, native.EPI_BF16),
    ("gate/up dgrad", 4096, 1024, 5632, False, True, native.EPI_BF16),
    ("qkv wgrad", 3072, 1024, 4096, True, True, native.EPI_F32),
    ("gate/up wgrad", 5632, 1024, 4096, True, True, native.EPI_F32),
    ("down wgrad", 1024, 2816, 4096, True, True, native.EPI_F32),
    ("o wgrad", 1024, 1024, 4096, True, True, native.EPI_F32),
    ("o dgrad", 4096, 1024, 1024, False, True, native.EPI_BF16),
    ("down dgrad", 4096, 2816, 1024, False, True, native.EPI_BF16),
    ("down dgrad+swiglu_bwd", 4096, 2816, 1024, False, True, native.EPI_SWIGLU_BWD),
    ("head wgrad", 32000, 1024, 4096, True, True, native.EPI_F32),
]


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    ap.add_argument("--no-cublas", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda")
    native.gemm_set_workspace(torch.empty(64 << 20, device=dev))
    res = []
    for name, M, N, K, a_mn, b_mn, epi in SHAPES:
        if a.only and a.only not in name:
            continue
        A = torch.randn((K, M) if a_mn else (M, K), device=dev).to(torch.bfloat16)
        B = torch.randn((K, N) if b_mn else (N, K), device=dev).to(torch.bfloat16)
        if epi == native.EPI_F32:
            C = torch.zeros(M, N, device=dev)
        elif epi == "rope":
            C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        elif epi == native.EPI_SWIGLU:
            C = torch.empty(M, N // 2, device=dev, dtype=torch.bfloat16)
        else:
            C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        C2 = torch.empty(M, N, device=dev, dtype=torch.bfloat16) if epi == native.EPI_SWIGLU else None
        R = torch.randn(M, N, device=dev).to(torch.bfloat16) if epi == native.EPI_BF16_RESID else None
        if epi == native.EPI_SWIGLU_BWD:  # R = gu [M, 2N] (gate/up interleave), C2 = dgu [M, 2N]
            R = torch.randn(M, 2 * N, device=dev).to(torch.bfloat16)
            C2 = torch.empty(M, 2 * N, device=dev, dtype=torch.bfloat16)
        ldc = N // 2 if epi == native.EPI_SWIGLU else N

        cs = torch.randn(32, 1024, 2, device=dev)

        def run():
            if epi == "rope":
                return native.gemm_rope(A, B, C, M=M, N=N, K=K, lda=K, ldb=K, ldc=N, cos_sin=cs, rope_cols=2048, T=1024,
                                        head_dim=64)
            native.gemm(A, B, C, M=M, N=N, K=K, lda=A.shape[1], ldb=B.shape[1], ldc=ldc, a_mn=a_mn, b_mn=b_mn,
                        epilogue=epi, R=R, C2=C2, ldc2=2 * N if epi == native.EPI_SWIGLU_BWD else N,
                        beta=1.0 if epi == native.EPI_F32 else 0.0)

        Am = A.t() if a_mn else A
        Bm = B.t() if b_mn else B

        def run_ref():
            torch.matmul(Am, Bm.t())

        out = {}
        out["cublas"] = (float("nan"), float("nan"))
        for label, fn in (("spx", run),) + (() if a.no_cublas else (("cublas", run_ref),)):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            # launches captured in a CUDA graph (as in the training step): no host overhead in the timing
            iters = 20
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(iters):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            g.replay()
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / iters
            out[label] = (ms, 2.0 * M * N * K / ms / 1e9)
        line = (f"{name:20s} M={M:6d} N={N:6d} K={K:6d}  spx {out['spx'][0]*1e3:8.1f} us "
                f"{out['spx'][1]:7.1f} TF/s | cublas {out['cublas'][0]*1e3:8.1f} us {out['cublas'][1]:7.1f} TF/s")
        print(line, flush=True)
        res.append(line)


if __name__ == "__main__":
    main()
