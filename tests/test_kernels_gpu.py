"""Stage kernels of libspx (attention, RMSNorm, RoPE, SwiGLU, embedding, cross-entropy, AdamW,
grad-norm) against plain torch fp32 references of the same ops."""

import math

import pytest
import torch

from paper_2502_19913_b200 import native

pytestmark = pytest.mark.gpu
dev = "cuda"


def rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-12)).item()


def bf(x):
    return x.to(torch.bfloat16)


def rope_table(T, hd, theta=10000.0):
    from paper_2502_19913_b200.model import rope_cos_sin

    return rope_cos_sin(T, hd, theta)  # [hd/2, T, 2], position-minor


def rope_ref(x, cs):  # x [B, T, H, hd] fp32; cs [hd/2, T, 2]
    hd = x.shape[-1]
    c = cs[..., 0].t()[None, :, None, :]
    s = cs[..., 1].t()[None, :, None, :]
    x1, x2 = x[..., : hd // 2], x[..., hd // 2:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def attn_ref(q, k, v, scale):  # [B, H, T, hd] fp32, causal, GQA by repeat
    rep = q.shape[1] // k.shape[1]
    k = k.repeat_interleave(rep, dim=1)
    v = v.repeat_interleave(rep, dim=1)
    s = (q @ k.transpose(-1, -2)) * scale
    T = q.shape[2]
    mask = torch.ones(T, T, dtype=torch.bool, device=q.device).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    return torch.softmax(s, dim=-1) @ v, lse


@pytest.mark.parametrize("B,T,H,Hkv,hd", [(2, 256, 6, 6, 48), (2, 1024, 16, 16, 64), (1, 512, 8, 2, 128),
                                          (1, 256, 4, 4, 128), (1, 4096, 8, 2, 128), (1, 2048, 4, 4, 64),
                                          (1, 128, 2, 2, 128), (3, 384, 4, 2, 128), (3, 384, 6, 3, 64),
                                          (1, 128, 2, 1, 64)])
def test_attention_fwd_bwd(B, T, H, Hkv, hd):
    g = torch.Generator().manual_seed(B * T + H + hd)
    W = (H + 2 * Hkv) * hd
    qkv = bf(torch.randn(B * T, W, generator=g)).to(dev)
    do = bf(torch.randn(B * T, H * hd, generator=g)).to(dev)
    scale = 1.0 / math.sqrt(hd)
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, H, T, dtype=torch.float32, device=dev)
    native.attn_fwd(qkv, o, lse, B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W, ld_o=H * hd, scale=scale)
    dqkv = torch.zeros_like(qkv)
    # sized with Hkv: GQA shapes with few kv-head tiles take the split dK/dV pass
    delta = torch.empty(native.attn_bwd_ws_floats(B, H, T, hd, Hkv), dtype=torch.float32, device=dev)
    native.attn_bwd(qkv, o, do, lse, delta, dqkv, B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W, ld_o=H * hd, scale=scale)
    torch.cuda.synchronize()

    x = qkv.float().view(B, T, H + 2 * Hkv, hd)
    q = x[:, :, :H].permute(0, 2, 1, 3).clone().requires_grad_()
    k = x[:, :, H:H + Hkv].permute(0, 2, 1, 3).clone().requires_grad_()
    v = x[:, :, H + Hkv:].permute(0, 2, 1, 3).clone().requires_grad_()
    ref, ref_lse = attn_ref(q, k, v, scale)
    ref.backward(do.float().view(B, T, H, hd).permute(0, 2, 1, 3))
    ref_o = ref.permute(0, 2, 1, 3).reshape(B * T, H * hd)
    assert rel(o, ref_o) < 1e-2
    assert (lse - ref_lse).abs().max().item() < 1e-2
    dx = dqkv.float().view(B, T, H + 2 * Hkv, hd)
    assert rel(dx[:, :, :H].permute(0, 2, 1, 3), q.grad) < 2e-2
    assert rel(dx[:, :, H:H + Hkv].permute(0, 2, 1, 3), k.grad) < 2e-2
    assert rel(dx[:, :, H + Hkv:].permute(0, 2, 1, 3), v.grad) < 2e-2


@pytest.mark.parametrize("q2", ["1", "0"])
def test_attention_forward_two_query_tiles(q2):
    """The hd=64 two-query-tile forward (forced on / off with SPX_ATTN_Q2, read once per process)
    against torch fp32 on shapes below and above its one-item-per-SM threshold, incl. GQA."""
    import os
    import subprocess
    import sys

    code = r'''
import math, torch
from paper_2502_19913_b200 import native
worst = 0.0
for (B, T, H, Hkv) in [(2, 1024, 16, 16), (1, 2048, 8, 2), (1, 512, 4, 4), (4, 1024, 16, 16)]:
    hd = 64
    g = torch.Generator().manual_seed(B * T + H)
    W = (H + 2 * Hkv) * hd
    qkv = torch.randn(B * T, W, generator=g).to(torch.bfloat16).cuda()
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B, H, T, device="cuda")
    native.attn_fwd(qkv, o, lse, B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W, ld_o=H * hd, scale=1 / math.sqrt(hd))
    x = qkv.float().view(B, T, H + 2 * Hkv, hd)
    q = x[:, :, :H].permute(0, 2, 1, 3)
    k = x[:, :, H:H + Hkv].permute(0, 2, 1, 3).repeat_interleave(H // Hkv, dim=1)
    v = x[:, :, H + Hkv:].permute(0, 2, 1, 3).repeat_interleave(H // Hkv, dim=1)
    sc = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
    sc = sc.masked_fill(torch.ones(T, T, dtype=torch.bool, device="cuda").triu(1), float("-inf"))
    ref = (torch.softmax(sc, -1) @ v).permute(0, 2, 1, 3).reshape(B * T, H * hd)
    rel = ((o.float() - ref).norm() / ref.norm()).item()
    lerr = (lse - torch.logsumexp(sc, -1)).abs().max().item()
    worst = max(worst, rel, lerr / 10)
print(worst)
'''
    env = dict(os.environ, SPX_ATTN_Q2=q2)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) < 1e-2


def test_attention_deterministic():
    B, T, H, hd = 1, 512, 4, 64
    g = torch.Generator().manual_seed(7)
    W = 3 * H * hd
    qkv = bf(torch.randn(B * T, W, generator=g)).to(dev)
    do = bf(torch.randn(B * T, H * hd, generator=g)).to(dev)
    outs = []
    for _ in range(2):
        o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(B, H, T, device=dev)
        native.attn_fwd(qkv, o, lse, B=B, T=T, H=H, Hkv=H, hd=hd, ld_qkv=W, ld_o=H * hd, scale=0.125)
        d = torch.zeros_like(qkv)
        native.attn_bwd(qkv, o, do, lse, torch.empty(native.attn_bwd_ws_floats(B, H, T, hd), device=dev), d, B=B, T=T, H=H, Hkv=H, hd=hd, ld_qkv=W,
                        ld_o=H * hd, scale=0.125)
        outs.append((o, d))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("rows,d,with_res", [(512, 288, True), (4096, 1024, True), (37, 256, False), (1000, 384, True),
                                              (300, 2048, True), (200, 4096, False), (130, 1024, False)])
def test_rmsnorm(rows, d, with_res):
    g = torch.Generator().manual_seed(d)
    x = bf(torch.randn(rows, d, generator=g)).to(dev)
    w = bf(1 + 0.1 * torch.randn(d, generator=g)).to(dev)
    dy = bf(torch.randn(rows, d, generator=g)).to(dev)
    dres = bf(torch.randn(rows, d, generator=g)).to(dev) if with_res else None
    y = torch.empty_like(x)
    rstd = torch.empty(rows, device=dev)
    native.rmsnorm_fwd(x, w, y, rstd, rows=rows, d=d, eps=1e-5)
    dx = torch.empty_like(x)
    dg = torch.full((d,), 0.5, device=dev)
    ws = torch.empty(native.rmsnorm_ws_floats(rows, d), device=dev)
    native.rmsnorm_bwd(x, w, rstd, dy, dres, dx, dg, ws, rows=rows, d=d)
    torch.cuda.synchronize()
    xr = x.float().requires_grad_()
    wr = w.float().requires_grad_()
    yr = xr * torch.rsqrt(xr.pow(2).mean(-1, keepdim=True) + 1e-5) * wr
    yr.backward(dy.float())
    assert rel(y, yr) < 1e-2
    assert rel(dx, xr.grad + (dres.float() if with_res else 0)) < 1e-2
    assert rel(dg - 0.5, wr.grad) < 1e-3
    # deterministic: a second backward gives identical bits
    dx2, dg2 = torch.empty_like(x), torch.full((d,), 0.5, device=dev)
    native.rmsnorm_bwd(x, w, rstd, dy, dres, dx2, dg2, ws, rows=rows, d=d)
    torch.cuda.synchronize()
    assert torch.equal(dx, dx2) and torch.equal(dg, dg2)


def test_rope_roundtrip():
    B, T, H, Hkv, hd = 2, 256, 4, 2, 64
    W = (H + 2 * Hkv) * hd
    g = torch.Generator().manual_seed(0)
    qkv = bf(torch.randn(B * T, W, generator=g)).to(dev)
    cs = rope_table(T, hd).to(dev)
    out = qkv.clone()
    native.rope(out, cs, rows=B * T, T=T, n_heads=H + Hkv, hd=hd, ld=W)
    torch.cuda.synchronize()
    x = qkv.float().view(B, T, H + 2 * Hkv, hd)
    ref = rope_ref(x[:, :, : H + Hkv], cs)
    assert rel(out.float().view(B, T, -1, hd)[:, :, : H + Hkv], ref) < 1e-2
    assert torch.equal(out.view(B, T, -1, hd)[:, :, H + Hkv:], qkv.view(B, T, -1, hd)[:, :, H + Hkv:])
    native.rope(out, cs, rows=B * T, T=T, n_heads=H + Hkv, hd=hd, ld=W, inverse=True)
    torch.cuda.synchronize()
    assert rel(out, qkv) < 2e-2


@pytest.mark.parametrize("rows,F", [(512, 768), (4096, 2816)])
def test_swiglu_bwd(rows, F):
    g = torch.Generator().manual_seed(F)
    gate = torch.randn(rows, F, generator=g)
    up = torch.randn(rows, F, generator=g)
    dh = bf(torch.randn(rows, F, generator=g)).to(dev)
    gu = torch.stack([gate.view(rows, F // 128, 128), up.view(rows, F // 128, 128)], dim=2).reshape(rows, 2 * F)
    gu = bf(gu).to(dev)
    dgu = torch.empty_like(gu)
    native.swiglu_bwd(gu, dh, dgu, rows=rows, F=F)
    torch.cuda.synchronize()
    gr = gu.float().view(rows, F // 128, 2, 128)
    gt = gr[:, :, 0].reshape(rows, F).requires_grad_()
    ut = gr[:, :, 1].reshape(rows, F).requires_grad_()
    (torch.nn.functional.silu(gt) * ut).backward(dh.float())
    d = dgu.float().view(rows, F // 128, 2, 128)
    assert rel(d[:, :, 0].reshape(rows, F), gt.grad) < 1e-2
    assert rel(d[:, :, 1].reshape(rows, F), ut.grad) < 1e-2


def test_embedding():
    V, d, n = 1000, 288, 512
    g = torch.Generator().manual_seed(0)
    table = bf(torch.randn(V, d, generator=g)).to(dev)
    ids_cpu = torch.randint(0, 50, (n,), generator=g, dtype=torch.int32)  # many repeats
    ids = ids_cpu.to(dev)
    out = torch.empty(n, d, dtype=torch.bfloat16, device=dev)
    native.embed_fwd(ids, table, out, n=n, d=d)
    dout = bf(torch.randn(n, d, generator=g)).to(dev)
    perm, seg, sid, nseg = native.embed_segments(ids_cpu)
    dtab = torch.zeros(V, d, device=dev)
    native.embed_bwd(perm.to(dev), seg.to(dev), sid.to(dev), nseg.to(dev), n, dout, dtab, d=d)
    torch.cuda.synchronize()
    assert torch.equal(out, table[ids.long()])
    ref = torch.zeros(V, d, device=dev).index_add_(0, ids.long(), dout.float())
    assert rel(dtab, ref) < 1e-5


@pytest.mark.parametrize("b,T,V,pad", [(1, 1, 7, 0), (2, 5, 3, 1), (4, 1024, 32000, 0), (3, 700, 50, 3),
                                       (1, 16384, 128256, 0), (16, 1024, 5, 0)])
@pytest.mark.parametrize("mode", ["fused", "split+group"])
def test_token_prep_matches_host_grouping(b, T, V, pad, mode):
    """Device token split + (id, position) grouping == the host reference, incl. heavy collisions,
    ragged n (not a power of two), row padding and the n = 16384 maximum; in one call, or as the
    executor issues it (split on one stream, grouping-only call after it)."""
    g = torch.Generator().manual_seed(b * 7 + T)
    tok = torch.randint(0, V, (b, T + 1 + pad), generator=g, dtype=torch.int64)
    n = b * T
    dt = tok.to(dev)
    ids, tgt, perm, sid = (torch.full((n,), -1, dtype=torch.int32, device=dev) for _ in range(4))
    seg = torch.full((n + 1,), -1, dtype=torch.int32, device=dev)
    nseg = torch.zeros(1, dtype=torch.int32, device=dev)
    if mode == "fused":
        native.token_prep(dt, ids, tgt, perm, seg, sid, nseg, b=b, T=T, ld=T + 1 + pad)
    else:
        native.token_prep(dt, ids, tgt, None, None, None, None, b=b, T=T, ld=T + 1 + pad)
        native.token_prep(dt, None, None, perm, seg, sid, nseg, b=b, T=T, ld=T + 1 + pad)
    torch.cuda.synchronize()
    ref_ids = tok[:, :T].reshape(-1).to(torch.int32)
    assert torch.equal(ids.cpu(), ref_ids)
    assert torch.equal(tgt.cpu(), tok[:, 1:T + 1].reshape(-1).to(torch.int32))
    rp, rs, ri, rn = native.embed_segments(ref_ids)
    k = int(rn.item())
    assert int(nseg.item()) == k
    assert torch.equal(perm.cpu(), rp)
    assert torch.equal(seg.cpu()[:k + 1], rs[:k + 1])
    assert torch.equal(sid.cpu()[:k], ri[:k])


def test_token_prep_rejects_oversize():
    t = torch.zeros(1, 16386, dtype=torch.int64, device=dev)
    z = torch.zeros(16386, dtype=torch.int32, device=dev)
    with pytest.raises(native.NativeError, match="16384"):
        native.token_prep(t, z, z, z, z, z, z, b=1, T=16385)


@pytest.mark.parametrize("n,V", [(512, 32000), (300, 1024)])
def test_xent(n, V):
    g = torch.Generator().manual_seed(V)
    z = bf(3 * torch.randn(n, V, generator=g)).to(dev)
    t = torch.randint(0, V, (n,), generator=g, dtype=torch.int32).to(dev)
    zz = z.clone()
    rl = torch.empty(n, device=dev)
    scale = 1.0 / n
    native.xent_fwd_bwd(zz, t, rl, n=n, V=V, ld=V, scale=scale)
    tot = torch.zeros(1, device=dev)
    native.sum_f32(rl, n, tot, scale=scale)
    torch.cuda.synchronize()
    zr = z.float().requires_grad_()
    loss = torch.nn.functional.cross_entropy(zr, t.long())
    loss.backward()
    assert abs(tot.item() - loss.item()) < 1e-3 * max(1, loss.item())
    assert rel(zz, zr.grad) < 1e-2


@pytest.mark.parametrize("n,V,d", [(512, 32000, 1024), (384, 128256, 256), (256, 384, 64)])
def test_head_gemm_xent_epilogue(n, V, d):
    """Head GEMM with the cross-entropy epilogue (EPI_XENT: logits + per-128-column (max, sum exp)
    partials) followed by spx_xent_from_parts equals torch fp32 cross-entropy on the same bf16
    logits, and the separate xent pass on the same logits (loss and dlogits)."""
    g = torch.Generator().manual_seed(V + d)
    x = bf(torch.randn(n, d, generator=g)).to(dev)
    w = bf(torch.randn(V, d, generator=g) * d ** -0.5 * 3).to(dev)
    t = torch.randint(0, V, (n,), generator=g, dtype=torch.int32).to(dev)
    nb = V // 128
    z = torch.empty(n, V, dtype=torch.bfloat16, device=dev)
    parts = torch.empty(n, 2 * nb, device=dev)
    native.gemm(x, w, z, M=n, N=V, K=d, lda=d, ldb=d, ldc=V, epilogue=native.EPI_XENT, C2=parts, ldc2=2 * nb)
    z_ref = z.clone()
    scale = 1.0 / n
    rl = torch.empty(n, device=dev)
    native.xent_from_parts(z, parts, t, rl, nb=nb, n=n, V=V, ld=V, scale=scale)
    rl2 = torch.empty(n, device=dev)
    z2 = z_ref.clone()
    native.xent_fwd_bwd(z2, t, rl2, n=n, V=V, ld=V, scale=scale)
    torch.cuda.synchronize()
    zr = z_ref.float().requires_grad_()
    loss = torch.nn.functional.cross_entropy(zr, t.long(), reduction="none")
    loss.sum().mul(scale).backward()
    assert (rl - loss.detach()).abs().max().item() < 1e-3 * max(1.0, loss.abs().max().item())
    assert (rl - rl2).abs().max().item() < 1e-4 * max(1.0, rl2.abs().max().item())
    assert rel(z, zr.grad) < 1e-2
    assert rel(z, z2) < 1e-2
    # inference form: loss only, logits untouched
    z3 = z_ref.clone()
    native.xent_from_parts(z3, parts, t, rl, nb=nb, n=n, V=V, ld=V, scale=0.0)
    torch.cuda.synchronize()
    assert torch.equal(z3, z_ref)


def test_adamw_and_clip():
    n, nd = 10_000, 7_000
    g = torch.Generator().manual_seed(0)
    p0 = torch.randn(n, generator=g)
    grads = [torch.randn(n, generator=g) * 3 for _ in range(3)]
    p = p0.clone().to(dev)
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    pb = torch.empty(n, dtype=torch.bfloat16, device=dev)
    ws = torch.empty(native.sumsq_ws_floats(), device=dev)
    ss = torch.empty(1, device=dev)
    sc = torch.empty(1, device=dev)
    # torch reference: two param groups (decay / no decay), clip_grad_norm_ 1.0
    pr1 = p0[:nd].clone().requires_grad_()
    pr2 = p0[nd:].clone().requires_grad_()
    opt = torch.optim.AdamW([{"params": [pr1], "weight_decay": 0.1}, {"params": [pr2], "weight_decay": 0.0}],
                            lr=3e-4, betas=(0.9, 0.95), eps=1e-8)
    for step, gr in enumerate(grads, start=1):
        gd = gr.to(dev)
        native.sumsq(gd, n, ws, ss)
        native.clip_scale(ss, 1, 1.0, sc)
        native.adamw(p, gd, m, v, pb, n=n, n_decay=nd, lr=3e-4, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1,
                     step=step, grad_scale=sc)
        pr1.grad, pr2.grad = gr[:nd].clone(), gr[nd:].clone()
        torch.nn.utils.clip_grad_norm_([pr1, pr2], 1.0)
        opt.step()
    torch.cuda.synchronize()
    ref = torch.cat([pr1.detach(), pr2.detach()])
    assert (p.cpu() - ref).abs().max().item() < 1e-6
    assert torch.equal(pb, p.to(torch.bfloat16))


def test_adamw_vector_path_bit_identical():
    """16-byte vector AdamW (aligned buffers) == scalar AdamW (buffers offset by one element)."""
    n, nd = 100_003, 61_001
    g = torch.Generator().manual_seed(1)
    base = [torch.randn(n + 1, generator=g).to(dev) for _ in range(2)]
    grad = (torch.randn(n + 1, generator=g) * 2).to(dev)
    sc = torch.full((1,), 0.7, device=dev)
    outs = []
    for off in (0, 1):  # off = 1 views every buffer at +4 bytes -> scalar kernel

        def place(t):
            buf = torch.empty(n + off, dtype=t.dtype, device=dev)
            buf[off:] = t
            return buf[off:]

        p, m, v = place(base[0][1:]), place(torch.zeros(n, device=dev)), place(base[1][1:].abs())
        pb, gg = place(torch.zeros(n, dtype=torch.bfloat16, device=dev)), place(grad[1:])
        assert (p.data_ptr() % 16 == 0) == (off == 0)
        for step in (1, 2, 3):
            native.adamw(p, gg, m, v, pb, n=n, n_decay=nd, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                         weight_decay=0.1, step=step, grad_scale=sc)
        torch.cuda.synchronize()
        outs.append((p.clone(), m.clone(), v.clone(), pb.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("hd,H,Hkv", [(64, 16, 16), (128, 8, 2)])
def test_gemm_rope_epilogue(hd, H, Hkv):
    B, T, d = 2, 256, 512
    g = torch.Generator().manual_seed(hd)
    W = (H + 2 * Hkv) * hd
    x = bf(torch.randn(B * T, d, generator=g) * 0.5).to(dev)
    w = bf(torch.randn(W, d, generator=g) * 0.05).to(dev)
    cs = rope_table(T, hd).to(dev)
    out = torch.empty(B * T, W, dtype=torch.bfloat16, device=dev)
    native.gemm_rope(x, w, out, M=B * T, N=W, K=d, lda=d, ldb=d, ldc=W, cos_sin=cs, rope_cols=(H + Hkv) * hd, T=T,
                     head_dim=hd)
    torch.cuda.synchronize()
    raw = (x.float() @ w.float().t()).view(B, T, H + 2 * Hkv, hd)
    ref = torch.cat([rope_ref(raw[:, :, : H + Hkv], cs), raw[:, :, H + Hkv:]], dim=2)
    assert rel(out.view(B, T, -1, hd), ref) < 1e-2


@pytest.mark.parametrize("hd,H,Hkv", [(64, 4, 4), (128, 4, 2)])
def test_attention_bwd_inverse_rope(hd, H, Hkv):
    B, T = 1, 256
    g = torch.Generator().manual_seed(11)
    W = (H + 2 * Hkv) * hd
    qkv = bf(torch.randn(B * T, W, generator=g)).to(dev)
    do = bf(torch.randn(B * T, H * hd, generator=g)).to(dev)
    cs = rope_table(T, hd).to(dev)
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, H, T, device=dev)
    native.attn_fwd(qkv, o, lse, B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W, ld_o=H * hd, scale=0.125)
    plain = torch.zeros_like(qkv)
    fused = torch.zeros_like(qkv)
    delta = torch.empty(native.attn_bwd_ws_floats(B, H, T, hd), device=dev)
    kw = dict(B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W, ld_o=H * hd, scale=0.125)
    native.attn_bwd(qkv, o, do, lse, delta, plain, **kw)
    native.attn_bwd(qkv, o, do, lse, delta, fused, rope_cs=cs, **kw)
    native.rope(plain, cs, rows=B * T, T=T, n_heads=H + Hkv, hd=hd, ld=W, inverse=True)
    torch.cuda.synchronize()
    assert rel(fused, plain) < 1e-2


@pytest.mark.parametrize("nbytes,ctas", [(16, 1), (4096 * 1024 * 2, 32), (294_912, 7), (1_000_000 - 1_000_000 % 16, 64)])
def test_hop_push_wait_bit_exact(nbytes, ctas):
    """spx_hop_push / spx_hop_wait (the cross-GPU hop, exercised here within one GPU): the copy
    is bit-exact for ragged sizes and CTA counts, every CTA adds 1 to the arrival flag, and the
    wait returns once the flag reaches its target."""
    src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev)
    dst = torch.zeros_like(src)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream()
    for rep in range(1, 4):
        native.hop_push(dst.data_ptr(), src, nbytes, flag.data_ptr(), ctas, stream=s)
        native.hop_wait(flag, rep * ctas, stream=s)
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    assert int(flag.item()) == 3 * ctas


def test_hop_push_ce_bit_exact():
    """spx_hop_push_ce (copy-engine hop + one flag increment), exercised within one GPU."""
    nbytes = 4096 * 1024 * 2
    src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev)
    dst = torch.zeros_like(src)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream()
    for rep in range(1, 4):
        native.hop_push_ce(dst.data_ptr(), src, nbytes, flag.data_ptr(), stream=s)
        native.hop_wait(flag, rep, stream=s)
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    assert int(flag.item()) == 3


@pytest.mark.parametrize("b,T,H,hd,d", [(2, 384, 4, 64, 512), (1, 256, 2, 128, 256), (4, 1024, 16, 64, 1024)])
def test_gemm_attn_delta_epilogue(b, T, H, hd, d):
    """spx_gemm_bf16_attn_delta: dO = dY . Wo plus the attention backward's D = rowsum(dO*O) and
    lse*log2e in the workspace prefix; the backward run with SPX_ATTN_DELTA_READY then matches the
    backward with its own D pass."""
    g = torch.Generator().manual_seed(b * T + hd)
    n, od = b * T, H * hd
    W = 3 * od
    dy = bf(torch.randn(n, d, generator=g)).to(dev)
    wo = bf(torch.randn(d, od, generator=g) / math.sqrt(d)).to(dev)
    qkv = bf(torch.randn(n, W, generator=g)).to(dev)
    o = torch.empty(n, od, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(b, H, T, device=dev)
    kw = dict(B=b, T=T, H=H, Hkv=H, hd=hd, ld_qkv=W, ld_o=od, scale=1 / math.sqrt(hd))
    native.attn_fwd(qkv, o, lse, **{k: v for k, v in kw.items()})
    do_ref = torch.empty(n, od, dtype=torch.bfloat16, device=dev)
    native.gemm(dy, wo, do_ref, M=n, N=od, K=d, lda=d, ldb=od, ldc=od, b_mn=True)
    do = torch.empty_like(do_ref)
    ws = torch.zeros(native.attn_bwd_ws_floats(b, H, T, hd), device=dev)
    native.gemm_attn_delta(dy, wo, do, o, lse, ws, M=n, N=od, K=d, lda=d, ldb=od, ldc=od, ld_o=od, batch=b, T=T,
                           head_dim=hd)
    ws_ref = torch.zeros_like(ws)
    d_ref, d_fused = torch.zeros_like(qkv), torch.zeros_like(qkv)
    native.attn_bwd(qkv, o, do_ref, lse, ws_ref, d_ref, **kw)
    native.attn_bwd(qkv, o, do, lse, ws, d_fused, delta_ready=True, **kw)
    torch.cuda.synchronize()
    assert torch.equal(do, do_ref)
    bht = b * H * T
    exact = (do.float().view(b, T, H, hd) * o.float().view(b, T, H, hd)).sum(-1).permute(0, 2, 1).reshape(-1)
    assert rel(ws[:bht], exact) < 1e-5
    assert rel(ws[:bht], ws_ref[:bht]) < 1e-5
    assert torch.equal(ws[bht:2 * bht], ws_ref[bht:2 * bht])
    assert rel(d_fused, d_ref) < 1e-3


@pytest.mark.parametrize("B,T,H,Hkv,hd", [(1, 1024, 32, 8, 128), (1, 512, 8, 2, 64), (2, 256, 8, 2, 128)])
def test_attention_bwd_gqa_split(B, T, H, Hkv, hd):
    """GQA backward with fewer (batch, kv head, key block) items than SMs: the split dK/dV pass
    (workspace sized by attn_bwd_ws_floats(..., Hkv), fp32 partials summed in a fixed order) agrees
    with the unsplit pass, is deterministic, and keeps dQ bit-identical; inverse RoPE included."""
    assert native.attn_bwd_ws_floats(B, H, T, hd, Hkv) > native.attn_bwd_ws_floats(B, H, T, hd)
    g = torch.Generator().manual_seed(T + H + hd)
    W = (H + 2 * Hkv) * hd
    qkv = bf(torch.randn(B * T, W, generator=g)).to(dev)
    do = bf(torch.randn(B * T, H * hd, generator=g)).to(dev)
    cs = rope_table(T, hd).to(dev)
    o = torch.empty(B * T, H * hd, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(B, H, T, device=dev)
    kw = dict(B=B, T=T, H=H, Hkv=Hkv, hd=hd, ld_qkv=W, ld_o=H * hd, scale=1 / math.sqrt(hd), rope_cs=cs)
    native.attn_fwd(qkv, o, lse, **{k: v for k, v in kw.items() if k != "rope_cs"})
    outs = []
    for hkv in (None, Hkv, Hkv):
        ws = torch.empty(native.attn_bwd_ws_floats(B, H, T, hd, hkv), device=dev)
        d = torch.zeros_like(qkv)
        native.attn_bwd(qkv, o, do, lse, ws, d, **kw)
        outs.append(d)
    torch.cuda.synchronize()
    plain, split, split2 = outs
    assert torch.equal(split, split2)
    assert torch.equal(split[:, :H * hd], plain[:, :H * hd])  # dQ untouched by the split
    assert rel(split[:, H * hd:], plain[:, H * hd:]) < 2e-3
