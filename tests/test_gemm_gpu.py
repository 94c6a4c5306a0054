"""tcgen05 GEMM (spx_gemm_bf16) against a plain torch fp32 reference of the same op."""

import pytest
import torch

from paper_2502_19913_b200 import native

pytestmark = pytest.mark.gpu

SHAPES = [
    (128, 256, 64),
    (256, 512, 128),
    (300, 288, 288),       # llama-50m: ragged M, N=d=288, K=288 (not a multiple of 64)
    (512, 864, 288),       # llama-50m QKV
    (4096, 3072, 1024),    # llama-500m QKV
    (4096, 1024, 2816),    # llama-500m down-proj (BN=128 path)
]


def _rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-12)).item()


def _mk(*shape, gen):
    return (torch.randn(*shape, generator=gen, device="cpu") * 0.5).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True), (True, False)])
def test_gemm_layouts(M, N, K, a_mn, b_mn):
    if (a_mn and M % 8) or (b_mn and N % 8):
        pytest.skip("TMA needs 16-byte row strides: MN-major operands need M/N % 8 == 0")
    g = torch.Generator().manual_seed(M * 7 + N + K)
    A = _mk(K, M, gen=g) if a_mn else _mk(M, K, gen=g)
    B = _mk(K, N, gen=g) if b_mn else _mk(N, K, gen=g)
    Am = A.float().t() if a_mn else A.float()
    Bm = B.float().t() if b_mn else B.float()
    ref = Am @ Bm.t()
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    native.gemm(A, B, C, M=M, N=N, K=K, lda=A.shape[1], ldb=B.shape[1], ldc=N, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    assert _rel(C, ref) < 1e-2


@pytest.mark.parametrize("M,N,K", [(300, 288, 288), (4096, 1024, 1024)])
def test_gemm_residual(M, N, K):
    g = torch.Generator().manual_seed(1)
    A, B, R = _mk(M, K, gen=g), _mk(N, K, gen=g), _mk(M, N, gen=g)
    ref = A.float() @ B.float().t() + R.float()
    native.gemm(A, B, R, M=M, N=N, K=K, lda=K, ldb=K, ldc=N, epilogue=native.EPI_BF16_RESID, R=R)
    torch.cuda.synchronize()
    assert _rel(R, ref) < 1e-2


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("M,N,K", [(288, 768, 512), (1024, 3072, 4096), (1024, 1024, 4096), (5632, 1024, 4096)])
def test_gemm_f32_accumulate(M, N, K, split):
    ws = torch.empty(8 * (M + 256) * N, device="cuda")
    native.gemm_set_workspace(ws if split else None)
    # wgrad form: dW[M=out,N=in] = dY^T X with both operands MN-major, accumulated twice.
    g = torch.Generator().manual_seed(2)
    dY, X = _mk(K, M, gen=g), _mk(K, N, gen=g)
    ref = 2.0 * (dY.float().t() @ X.float())
    C = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    for beta in (0.0, 1.0):
        native.gemm(dY, X, C, M=M, N=N, K=K, lda=M, ldb=N, ldc=N, a_mn=True, b_mn=True,
                    epilogue=native.EPI_F32, beta=beta)
    torch.cuda.synchronize()
    native.gemm_set_workspace(None)
    assert _rel(C, ref) < 5e-3


@pytest.mark.parametrize("epi", ["f32", "bf16"])
def test_gemm_n_major_raster(epi):
    """A multi-wave grid whose A operand exceeds the L2 budget walks N first (pick_raster): the
    LM-head weight-gradient form (large M, small N) and a K-major bf16 product of the same shape."""
    M, N, K = 16384, 512, 2048
    g = torch.Generator().manual_seed(5)
    if epi == "f32":
        A, B = _mk(K, M, gen=g), _mk(K, N, gen=g)
        ref = A.float().t() @ B.float()
        C = torch.zeros(M, N, dtype=torch.float32, device="cuda")
        native.gemm(A, B, C, M=M, N=N, K=K, lda=M, ldb=N, ldc=N, a_mn=True, b_mn=True, epilogue=native.EPI_F32,
                    beta=1.0)
    else:
        A, B = _mk(M, K, gen=g), _mk(N, K, gen=g)
        ref = A.float() @ B.float().t()
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        native.gemm(A, B, C, M=M, N=N, K=K, lda=K, ldb=K, ldc=N)
    torch.cuda.synchronize()
    assert _rel(C, ref) < 1e-2


def test_gemm_split_k_deterministic():
    M, N, K = 1024, 1024, 4096
    g = torch.Generator().manual_seed(9)
    dY, X = _mk(K, M, gen=g), _mk(K, N, gen=g)
    native.gemm_set_workspace(torch.empty(8 * (M + 256) * N, device="cuda"))
    outs = []
    for _ in range(3):
        C = torch.zeros(M, N, dtype=torch.float32, device="cuda")
        native.gemm(dY, X, C, M=M, N=N, K=K, lda=M, ldb=N, ldc=N, a_mn=True, b_mn=True, epilogue=native.EPI_F32,
                    beta=1.0)
        outs.append(C)
    torch.cuda.synchronize()
    native.gemm_set_workspace(None)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])


@pytest.mark.parametrize("M,F,K", [(512, 768, 288), (4096, 2816, 1024)])
def test_gemm_swiglu(M, F, K):
    g = torch.Generator().manual_seed(3)
    X = _mk(M, K, gen=g)
    Wg, Wu = _mk(F, K, gen=g), _mk(F, K, gen=g)
    # 128-row interleave: [g0..g127, u0..u127, g128.., u128..]
    W = torch.stack([Wg.view(F // 128, 128, K), Wu.view(F // 128, 128, K)], dim=1).reshape(2 * F, K).contiguous()
    H = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    GU = torch.empty(M, 2 * F, dtype=torch.bfloat16, device="cuda")
    native.gemm(X, W, H, M=M, N=2 * F, K=K, lda=K, ldb=K, ldc=F, epilogue=native.EPI_SWIGLU, C2=GU, ldc2=2 * F)
    torch.cuda.synchronize()
    gate = X.float() @ Wg.float().t()
    up = X.float() @ Wu.float().t()
    ref = torch.nn.functional.silu(gate) * up
    assert _rel(H, ref) < 2e-2
    gu = GU.view(M, F // 128, 2, 128)
    assert _rel(gu[:, :, 0].reshape(M, F), gate) < 1e-2
    assert _rel(gu[:, :, 1].reshape(M, F), up) < 1e-2


@pytest.mark.parametrize("M,F,K", [(512, 768, 288), (4096, 2816, 1024)])
def test_gemm_swiglu_bwd_epilogue(M, F, K):
    """dh = dy . Wdown with the SwiGLU backward fused: dgu vs torch autograd of silu(g)*u."""
    g = torch.Generator().manual_seed(5)
    dy = _mk(M, K, gen=g)                      # grad of the down-projection output, K = d
    wd = _mk(K, F, gen=g)                      # Wdown [d, F]
    gate, up = torch.randn(M, F, generator=g), torch.randn(M, F, generator=g)
    gu = torch.stack([gate.view(M, F // 128, 128), up.view(M, F // 128, 128)], dim=2).reshape(M, 2 * F)
    gu = gu.to(torch.bfloat16).cuda()
    dgu = torch.empty_like(gu)
    native.gemm(dy, wd, None, M=M, N=F, K=K, lda=K, ldb=F, ldc=F, b_mn=True, epilogue=native.EPI_SWIGLU_BWD, R=gu,
                C2=dgu, ldc2=2 * F)
    torch.cuda.synchronize()
    dh = dy.float() @ wd.float()
    gr = gu.float().view(M, F // 128, 2, 128)
    gt = gr[:, :, 0].reshape(M, F).requires_grad_()
    ut = gr[:, :, 1].reshape(M, F).requires_grad_()
    (torch.nn.functional.silu(gt) * ut).backward(dh)
    d = dgu.float().view(M, F // 128, 2, 128)
    assert _rel(d[:, :, 0].reshape(M, F), gt.grad) < 2e-2
    assert _rel(d[:, :, 1].reshape(M, F), ut.grad) < 2e-2


@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_gemm_f32_group(beta):
    """Four wgrad-shaped problems (incl. ragged M/N) in one grouped launch == four torch matmuls."""
    g = torch.Generator().manual_seed(11)
    shapes = [(768, 256, 512), (288, 512, 512), (1024, 2816, 1024), (320, 96, 1024)]
    probs, refs = [], []
    for (M, N, K) in shapes:
        dY, X = _mk(K, M, gen=g), _mk(K, N, gen=g)
        C = torch.randn(M, N, generator=g).cuda()
        refs.append(beta * C + dY.float().t() @ X.float())
        probs.append(dict(A=dY, B=X, C=C, M=M, N=N, K=K, lda=M, ldb=N, ldc=N, beta=beta))
    native.gemm_f32_group(probs)
    torch.cuda.synchronize()
    for p, ref in zip(probs, refs):
        assert _rel(p["C"], ref) < 5e-3
    # one problem alone equals the single-GEMM path bit for bit
    C1 = torch.zeros(768, 256, device="cuda")
    C2 = torch.zeros(768, 256, device="cuda")
    p0 = dict(probs[0], C=C1, beta=0.0)
    native.gemm_f32_group([p0])
    native.gemm(p0["A"], p0["B"], C2, M=768, N=256, K=512, lda=768, ldb=256, ldc=256, a_mn=True, b_mn=True,
                epilogue=native.EPI_F32)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2)


def test_gemm_f32_group_large_m():
    """Grouped wgrad launch with every M > 512 (ragged M and N) and a large plain GEMM == torch."""
    g = torch.Generator().manual_seed(5)
    shapes = [(1280, 256, 512), (800, 512, 256), (1024, 288, 256), (1536, 96, 512)]
    probs, refs = [], []
    for (M, N, K) in shapes:
        dY, X = _mk(K, M, gen=g), _mk(K, N, gen=g)
        C = torch.randn(M, N, generator=g).cuda()
        refs.append(C + dY.float().t() @ X.float())
        probs.append(dict(A=dY, B=X, C=C, M=M, N=N, K=K, lda=M, ldb=N, ldc=N, beta=1.0))
    native.gemm_f32_group(probs)
    torch.cuda.synchronize()
    for p, ref in zip(probs, refs):
        assert _rel(p["C"], ref) < 5e-3
