"""Time the softmax cross-entropy kernel at the C2 head shape (4096 x 32000 bf16 logits)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19913_b200 import native  # noqa: E402

n, V = 4096, 32000
z = torch.randn(n, V, device="cuda").to(torch.bfloat16)
t = torch.randint(0, V, (n,), device="cuda", dtype=torch.int32)
rl = torch.empty(n, device="cuda")
zz = z.clone()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    native.xent_fwd_bwd(zz, t, rl, n=n, V=V, ld=V, scale=1.0 / n, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            native.xent_fwd_bwd(zz, t, rl, n=n, V=V, ld=V, scale=1.0 / n, stream=s)
    g.replay()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    s.synchronize()
tot = e0.elapsed_time(e1) / 10 * 1e3
print(f"xent {tot:.1f} us per launch, {2 * n * V * 2 / tot / 1e3:.0f} GB/s (262 MB read + 262 MB write)")
