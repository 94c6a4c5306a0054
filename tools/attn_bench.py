"""Time spx_attn_fwd / spx_attn_bwd at the C2 (and C3) shapes with CUDA events."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19913_b200 import native  # noqa: E402
from paper_2502_19913_b200.model import rope_cos_sin  # noqa: E402


def bench(B, T, H, Hkv, hd, iters=20):
    W = (H + 2 * Hkv) * hd
    qkv = (torch.randn(B * T, W, device="cuda") * 0.5).to(torch.bfloat16)
    do = torch.randn(B * T, H * hd, device="cuda").to(torch.bfloat16)
    o = torch.empty(B * T, H * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, H, T, device="cuda")
    dq = torch.empty_like(qkv)
    delta = torch.empty(native.attn_bwd_ws_floats(B, H, T, hd), device="cuda")
    cs = rope_cos_sin(T, hd, 10000.0).cuda()
    sc = 1 / math.sqrt(hd)
    f = lambda: native.attn_fwd(qkv, o, lse, B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W, ld_o=H * hd, scale=sc)  # noqa
    bw = lambda: native.attn_bwd(qkv, o, do, lse, delta, dq, B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W,  # noqa
                                 ld_o=H * hd, scale=sc, rope_cs=cs)
    out = []
    for fn in (f, bw):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / iters * 1e3)
    fl = 4 * B * H * T * T / 2 * hd
    print(f"B={B} T={T} H={H} Hkv={Hkv} hd={hd}: fwd {out[0]:.1f} us ({fl / out[0] / 1e6:.0f} TF/s)  "
          f"bwd {out[1]:.1f} us ({2.5 * fl / out[1] / 1e6:.0f} TF/s)", flush=True)


if __name__ == "__main__":
    bench(4, 1024, 16, 16, 64)
    bench(1, 4096, 16, 16, 64)
    bench(16, 1024, 16, 16, 64)
    bench(1, 4096, 16, 16, 128)
    bench(1, 4096, 32, 8, 128)
