"""One C2-shaped attention fwd+bwd (for ncu captures)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2502_19913_b200 import native  # noqa: E402
from paper_2502_19913_b200.model import rope_cos_sin  # noqa: E402
B, T, H, hd = 4, 1024, 16, 64
W = 3 * H * hd
qkv = (torch.randn(B * T, W, device="cuda") * 0.5).to(torch.bfloat16)
do = torch.randn(B * T, H * hd, device="cuda").to(torch.bfloat16)
o = torch.empty(B * T, H * hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B, H, T, device="cuda")
dq = torch.empty_like(qkv)
delta = torch.empty(native.attn_bwd_ws_floats(B, H, T, hd), device="cuda")
cs = rope_cos_sin(T, hd, 10000.0).cuda()
for _ in range(3):
    native.attn_fwd(qkv, o, lse, B=B, T=T, H=H, Hkv=H, hd=hd, ld_qkv=W, ld_o=H * hd, scale=0.125)
    native.attn_bwd(qkv, o, do, lse, delta, dq, B=B, T=T, H=H, Hkv=H, hd=hd, ld_qkv=W, ld_o=H * hd, scale=0.125,
                    rope_cs=cs)
torch.cuda.synchronize()
print("ok")
