"""tcgen05 GEMM (p2r_gemm) vs a plain PyTorch fp32 matmul of the same bf16 operands.

Covers the three layouts the training step uses (forward X.W, dX = dY.W^T,
dW = X^T.dY), every fused epilogue, ragged M/N, split-K and the grouped
(MoE expert) variants.
"""
import ctypes

import pytest

pytestmark = pytest.mark.gpu


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _run(args):
    import torch
    from paper_2110_03888_b200 import _lib
    st = _lib.lib().p2r_gemm(ctypes.byref(args), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _lib.check(st)
    torch.cuda.synchronize()


def _args(**kw):
    from paper_2110_03888_b200._lib import GemmArgs
    a = GemmArgs()
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def _rel(x, y):
    return float((x.float() - y.float()).norm() / (y.float().norm() + 1e-30))


@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (1024, 1024, 1024), (1000, 260, 256), (8192, 3072, 1024), (77, 40, 200)])
def test_gemm_kk_f32_bias_resid(cuda, m, n, k):
    import torch
    from paper_2110_03888_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = torch.randn(n, k, device=cuda, generator=g).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g)
    ldc = (n + 7) // 8 * 8
    R = torch.randn(m, ldc, device=cuda, generator=g)
    C = torch.empty(m, ldc, device=cuda)
    _run(_args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_F32,
               c=_ptr(C), ldc=ldc, bias=_ptr(bias), aux=_ptr(R), ldaux=ldc, split_k=1))
    ref = A.float() @ B.float().T + bias + R[:, :n]
    assert _rel(C[:, :n], ref) < 1e-5


def dgelu(x):
    """exact-erf GELU derivative (tensor.cpp:249-260)"""
    import torch
    return 0.5 * (1 + torch.erf(x / 2 ** 0.5)) + x * torch.exp(-0.5 * x * x) / (2 * torch.pi) ** 0.5


@pytest.mark.parametrize("m,n,k", [(256, 512, 128), (8192, 4096, 1024)])
def test_gemm_bias_gelu_and_dgelu(cuda, m, n, k):
    import torch
    from paper_2110_03888_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = (0.05 * torch.randn(n, k, device=cuda, generator=g)).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g) * 0.1
    G = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    H = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    _run(_args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_BIAS_GELU,
               c=_ptr(G), ldc=n, c2=_ptr(H), ldc2=n, bias=_ptr(bias), split_k=1))
    pre = A.float() @ B.float().T + bias
    assert _rel(H, dgelu(pre)) < 8e-3  # the stored GELU derivative
    assert _rel(G, torch.nn.functional.gelu(pre)) < 8e-3
    # DGELU: D = (A.B^T) * H (the stored derivative)
    D = torch.empty(m, n, device=cuda, dtype=torch.bfloat16)
    _run(_args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_DGELU,
               c=_ptr(D), ldc=n, aux=_ptr(H), ldaux=n, split_k=1))
    ref = (A.float() @ B.float().T) * H.float()
    assert _rel(D, ref) < 8e-3


@pytest.mark.parametrize("m,n,ldc,k", [(1000, 264, 264, 320), (300, 520, 528, 128), (130, 260, 260, 64),
                                       (8192, 3072, 3072, 1024)])
def test_gemm_bf16_epilogues_ragged(cuda, m, n, ldc, k):
    """bf16 / bias+GELU / GELU' outputs with partial row tiles and column chunks: the
    TMA-store epilogue (ldc % 8 == 0) clips at the edges and leaves padding columns
    untouched; ldc % 8 != 0 takes the per-thread store path."""
    import torch
    from paper_2110_03888_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = (0.1 * torch.randn(n, k, device=cuda, generator=g)).bfloat16()
    bias = torch.randn(n, device=cuda, generator=g) * 0.1
    acc = A.float() @ B.float().T
    Y = torch.full((m, ldc), 3.0, device=cuda).bfloat16()
    _run(_args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_BF16, c=_ptr(Y), ldc=ldc,
               bias=_ptr(bias), split_k=1))
    assert _rel(Y[:, :n], acc + bias) < 8e-3
    assert bool((Y[:, n:] == 3.0).all())
    G = torch.full((m, ldc), 3.0, device=cuda).bfloat16()
    H = torch.full((m, ldc), 3.0, device=cuda).bfloat16()
    _run(_args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_BIAS_GELU, c=_ptr(G), ldc=ldc,
               c2=_ptr(H), ldc2=ldc, bias=_ptr(bias), split_k=1))
    assert _rel(H[:, :n], dgelu(acc + bias)) < 8e-3
    assert _rel(G[:, :n], torch.nn.functional.gelu(acc + bias)) < 8e-3
    assert bool((G[:, n:] == 3.0).all()) and bool((H[:, n:] == 3.0).all())
    D = torch.full((m, ldc), 3.0, device=cuda).bfloat16()
    _run(_args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_DGELU, c=_ptr(D), ldc=ldc,
               aux=_ptr(H), ldaux=ldc, split_k=1))
    assert _rel(D[:, :n], acc * H[:, :n].float()) < 8e-3
    assert bool((D[:, n:] == 3.0).all())


@pytest.mark.parametrize("m,n,ldc,k", [(8192, 4096, 4096, 1024), (1000, 264, 264, 320), (77, 130, 136, 64)])
def test_gemm_dgelu_bias_grad(cuda, m, n, ldc, k):
    """GELU' with bias_grad: the epilogue's per-32-row column partials of the fp32
    GELU' output (before its bf16 rounding, as the reference's fp32 colsum) + the
    finish kernel add the column sums into bias_grad."""
    import torch
    from paper_2110_03888_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(6)
    A = torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = (0.1 * torch.randn(n, k, device=cuda, generator=g)).bfloat16()
    H = torch.randn(m, ldc, device=cuda, generator=g).bfloat16()
    D = torch.empty(m, ldc, device=cuda).bfloat16()
    db0 = torch.randn(n, device=cuda, generator=g)
    db = db0.clone()
    args = _args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_DGELU, c=_ptr(D), ldc=ldc,
                 aux=_ptr(H), ldaux=ldc, split_k=1, bias_grad=_ptr(db))
    ws_bytes = _lib.lib().p2r_gemm_workspace_bytes(ctypes.byref(args))
    assert ws_bytes == (m + 31) // 32 * n * 4
    ws = torch.empty(ws_bytes // 4, device=cuda)
    _lib.check(_lib.lib().p2r_set_workspace(_ptr(ws), ws_bytes))
    _run(args)
    dg = H[:, :n].float()  # aux = the stored GELU derivative
    assert _rel(D[:, :n], (A.float() @ B.float().T) * dg) < 8e-3
    terms = (A.double() @ B.double().T) * dg.double()
    ref = db0.double() + terms.sum(0)
    assert bool(((db.double() - ref).abs() <= 1e-5 * terms.abs().sum(0) + 1e-6).all())
    with pytest.raises(Exception, match="bias_grad"):
        bad = _args(m=m, n=n, k=k, a=_ptr(A), lda=k, b=_ptr(B), ldb=k, epi=_lib.EPI_BF16, c=_ptr(D), ldc=ldc,
                    split_k=1, bias_grad=_ptr(db))
        _run(bad)


@pytest.mark.parametrize("m,n,k,split", [(1024, 1024, 8192, 1), (1024, 3072, 8192, 4), (256, 260, 1024, 2), (200, 136, 1000, 3)])
def test_gemm_mn_major_acc(cuda, m, n, k, split):
    """dW += X^T . dY with both operands token-major (MN-major) and beta=1."""
    import torch
    from paper_2110_03888_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(2)
    lda = (m + 7) // 8 * 8
    ldb = (n + 7) // 8 * 8
    X = torch.randn(k, lda, device=cuda, generator=g).bfloat16()
    dY = torch.randn(k, ldb, device=cuda, generator=g).bfloat16()
    W0 = torch.randn(m, n, device=cuda, generator=g)
    C = W0.clone()
    args = _args(m=m, n=n, k=k, a=_ptr(X), lda=lda, a_mn_major=1, b=_ptr(dY), ldb=ldb, b_mn_major=1,
                 epi=_lib.EPI_ACC_F32, c=_ptr(C), ldc=n, split_k=split)
    ws_bytes = _lib.lib().p2r_gemm_workspace_bytes(ctypes.byref(args))
    ws = torch.empty(max(ws_bytes // 4, 1), device=cuda)
    _lib.check(_lib.lib().p2r_set_workspace(_ptr(ws), ws_bytes))
    _run(args)
    ref = W0 + X[:, :m].float().T @ dY[:, :n].float()
    assert _rel(C, ref) < 1e-5


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 8192), (1024, 3072, 8192), (4096, 1024, 8192), (260, 1024, 8192),
                                   (200, 136, 4000), (1000, 600, 3000)])
def test_gemm_acc_auto_split(cuda, m, n, k):
    """Auto split (split_k = 0) of C += A^T.B: wide splits accumulate in place in
    split order (tile counters), narrow ones go through partials + reduce. Three
    back-to-back launches reuse the counters; the result is bitwise stable."""
    import torch
    from paper_2110_03888_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(3)
    lda, ldb = (m + 7) // 8 * 8, (n + 7) // 8 * 8
    X = torch.randn(k, lda, device=cuda, generator=g).bfloat16()
    dY = torch.randn(k, ldb, device=cuda, generator=g).bfloat16()
    W0 = torch.randn(m, n, device=cuda, generator=g)
    outs = []
    for _ in range(2):
        C = W0.clone()
        args = _args(m=m, n=n, k=k, a=_ptr(X), lda=lda, a_mn_major=1, b=_ptr(dY), ldb=ldb, b_mn_major=1,
                     epi=_lib.EPI_ACC_F32, c=_ptr(C), ldc=n, split_k=0)
        ws_bytes = _lib.lib().p2r_gemm_workspace_bytes(ctypes.byref(args))
        ws = torch.empty(max(ws_bytes // 4, 1), device=cuda)
        _lib.check(_lib.lib().p2r_set_workspace(_ptr(ws), ws_bytes))
        for _ in range(3):
            _run(args)
        outs.append(C)
    ref = W0 + 3 * (X[:, :m].float().T @ dY[:, :n].float())
    assert _rel(outs[0], ref) < 1e-5
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("amn,bmn", [(0, 1), (1, 0)])
def test_gemm_mixed_major(cuda, amn, bmn):
    import torch
    from paper_2110_03888_b200 import _lib
    m, n, k = 512, 384, 320
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(k, m, device=cuda, generator=g).bfloat16() if amn else torch.randn(m, k, device=cuda, generator=g).bfloat16()
    B = torch.randn(k, n, device=cuda, generator=g).bfloat16() if bmn else torch.randn(n, k, device=cuda, generator=g).bfloat16()
    C = torch.empty(m, n, device=cuda)
    _run(_args(m=m, n=n, k=k, a=_ptr(A), lda=A.shape[1], a_mn_major=amn, b=_ptr(B), ldb=B.shape[1],
               b_mn_major=bmn, epi=_lib.EPI_F32, c=_ptr(C), ldc=n, split_k=1))
    Af = A.float().T if amn else A.float()
    Bf = B.float() if bmn else B.float().T
    assert _rel(C, Af @ Bf) < 1e-5


def test_gemm_grouped(cuda):
    """Expert GEMMs: GROUP_M forward (per-expert weights) and GROUP_K weight grads."""
    import torch
    from paper_2110_03888_b200 import _lib
    E, seg, d, f = 4, 384, 256, 512
    counts = torch.tensor([300, 0, 129, 384], device=cuda, dtype=torch.int32)
    g = torch.Generator(device="cuda").manual_seed(4)
    X = torch.zeros(E * seg, d, device=cuda).bfloat16()
    for e in range(E):
        c = int(counts[e])
        X[e * seg:e * seg + c] = torch.randn(c, d, device=cuda, generator=g).bfloat16()
    W = (0.05 * torch.randn(E, f, d, device=cuda, generator=g)).bfloat16()  # [E, N, K]
    bias = torch.randn(E, f, device=cuda, generator=g)
    H = torch.full((E * seg, f), 7.0, device=cuda).bfloat16()
    Hp = torch.full((E * seg, f), 7.0, device=cuda).bfloat16()
    _run(_args(m=E * seg, n=f, k=d, a=_ptr(X), lda=d, b=_ptr(W), ldb=d, epi=_lib.EPI_BIAS_GELU,
               c=_ptr(H), ldc=f, c2=_ptr(Hp), ldc2=f, bias=_ptr(bias), group_mode=_lib.GROUP_M,
               groups=E, seg_rows=seg, counts=_ptr(counts), split_k=1))
    for e in range(E):
        c = int(counts[e])
        pre = X[e * seg:e * seg + c].float() @ W[e].float().T + bias[e]
        if c:
            assert _rel(Hp[e * seg:e * seg + c], dgelu(pre)) < 8e-3
            assert _rel(H[e * seg:e * seg + c], torch.nn.functional.gelu(pre)) < 8e-3
        # padding rows inside a touched tile are zeroed
        top = min(seg, (c + 127) // 128 * 128)
        if top > c:
            assert float(H[e * seg + c:e * seg + top].float().abs().max()) == 0.0
    # GROUP_K: dW_e += X_e^T . H_e
    dW = torch.randn(E, d, f, device=cuda, generator=g)
    dW0 = dW.clone()
    _run(_args(m=d, n=f, k=seg, a=_ptr(X), lda=d, a_mn_major=1, b=_ptr(H), ldb=f, b_mn_major=1,
               epi=_lib.EPI_ACC_F32, c=_ptr(dW), ldc=f, group_mode=_lib.GROUP_K, groups=E,
               seg_rows=seg, counts=_ptr(counts), split_k=1))
    for e in range(E):
        c = int(counts[e])
        ref = dW0[e] + X[e * seg:e * seg + c].float().T @ H[e * seg:e * seg + c].float()
        assert _rel(dW[e], ref) < 1e-5
