"""Graph-replayed timings of the C2 per-layer elementwise kernels (RMSNorm fwd/bwd, SwiGLU bwd) with
their algorithmic bytes, warm (inputs just written, as inside a layer) and cold (L2 flushed).

    python tools/ew_bench.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19913_b200 import native  # noqa: E402

rows, d, F = 4096, 1024, 2816
dev = "cuda"
bf = dict(dtype=torch.bfloat16, device=dev)
x, dy, dres, dx = (torch.randn(rows, d, **bf) for _ in range(4))
g = torch.ones(d, **bf)
y = torch.empty(rows, d, **bf)
rstd = torch.empty(rows, device=dev)
dg = torch.zeros(d, device=dev)
ws = torch.empty(native.rmsnorm_ws_floats(rows, d), device=dev)
gu = torch.randn(rows, 2 * F, **bf)
dh = torch.randn(rows, F, **bf)
dgu = torch.empty(rows, 2 * F, **bf)
flush = torch.empty(256 * 1024 * 1024 // 4, device=dev)

cases = {
    "rmsnorm_fwd": (lambda s: native.rmsnorm_fwd(x, g, y, rstd, rows=rows, d=d, eps=1e-5, stream=s), 2 * rows * d * 2),
    "rmsnorm_bwd": (lambda s: native.rmsnorm_bwd(x, g, rstd, dy, dres, dx, dg, ws, rows=rows, d=d, stream=s),
                    4 * rows * d * 2),
    "swiglu_bwd": (lambda s: native.swiglu_bwd(gu, dh, dgu, rows=rows, F=F, stream=s), 5 * rows * F * 2),
}
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for name, (fn, nbytes) in cases.items():
        out = []
        for cold in (False, True):
            fn(s)
            s.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                if cold:
                    flush.zero_()
                fn(s)
            gr.replay()
            s.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(s)
            for _ in range(20):
                gr.replay()
            ev[1].record(s)
            s.synchronize()
            t = ev[0].elapsed_time(ev[1]) / 20 * 1e3
            if cold:  # subtract the flush itself
                gf = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gf, stream=s):
                    flush.zero_()
                ev[0].record(s)
                for _ in range(20):
                    gf.replay()
                ev[1].record(s)
                s.synchronize()
                t -= ev[0].elapsed_time(ev[1]) / 20 * 1e3
            out.append(t)
        print(f"{name:12s} warm {out[0]:6.1f} us ({nbytes / out[0] / 1e3:5.0f} GB/s)   "
              f"cold {out[1]:6.1f} us ({nbytes / out[1] / 1e3:5.0f} GB/s)")
