"""Per-block timestamps (clock64) of CTA 0 of the attention forward (SPX_ATTN_PROBE=<file>).

    SPX_ATTN_PROBE=/tmp/fa.bin python tools/attn_probe.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_19913_b200 import native  # noqa: E402

B, T, H, hd = 4, 1024, 16, 64
W = 3 * H * hd
qkv = (torch.randn(B * T, W, device="cuda") * 0.5).to(torch.bfloat16)
o = torch.empty(B * T, H * hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B, H, T, device="cuda")
for _ in range(5):
    native.attn_fwd(qkv, o, lse, B=B, T=T, H=H, Hkv=H, hd=hd, ld_qkv=W, ld_o=H * hd, scale=0.125)
torch.cuda.synchronize()
a = np.fromfile(os.environ["SPX_ATTN_PROBE"], dtype=np.uint64).reshape(3, 64, 8).astype(np.int64)
t0 = a[0, 0, 0]
n = int(((a[1, :, 0] > 0) | (a[2, :, 0] > 0)).sum())
print("blocks", n)
for g in range(min(n, 24)):
    row = lambda v: " ".join(f"{(x - t0) if x else -1:6d}" for x in v)  # noqa: E731
    print(f"{g:2d} MMA {row(a[0, g, :6])} | WG0 {row(a[1, g, :6])} | WG1 {row(a[2, g, :6])}")
