import ctypes, sys, torch
sys.path.insert(0, ".")
from paper_2110_03888_b200 import _lib
cuda = torch.device("cuda")
E, seg, d, f = 4, 384, 256, 512
counts = torch.tensor([300, 0, 129, 384], device=cuda, dtype=torch.int32)
X = torch.zeros(E * seg, d, device=cuda).bfloat16()
for e in range(E):
    c = int(counts[e]); X[e*seg:e*seg+c] = torch.randn(c, d, device=cuda).bfloat16()
W = (0.05 * torch.randn(E, f, d, device=cuda)).bfloat16()
for use_bias in (0, 1):
    bias = torch.randn(E, f, device=cuda)
    H = torch.full((E * seg, f), 7.0, device=cuda).bfloat16()
    Hp = torch.full((E * seg, f), 7.0, device=cuda).bfloat16()
    a = _lib.GemmArgs(m=E*seg, n=f, k=d, a=X.data_ptr(), lda=d, b=W.data_ptr(), ldb=d, epi=_lib.EPI_BIAS_GELU,
        c=H.data_ptr(), ldc=f, c2=Hp.data_ptr(), ldc2=f, bias=bias.data_ptr() if use_bias else None,
        group_mode=_lib.GROUP_M, groups=E, seg_rows=seg, counts=counts.data_ptr(), split_k=1)
    _lib.check(_lib.lib().p2r_gemm(ctypes.byref(a), torch.cuda.current_stream().cuda_stream)); torch.cuda.synchronize()
    for e in range(E):
        c = int(counts[e])
        if not c: continue
        pre = X[e*seg:e*seg+c].float() @ W[e].float().T + (bias[e] if use_bias else 0)
        got = Hp[e*seg:e*seg+c].float()
        err = (got - pre).abs()
        print("bias", use_bias, "e", e, "rel", float((got-pre).norm()/pre.norm()), "bad rows", int((err.max(1).values > 0.05).sum()), "bad cols", int((err.max(0).values > 0.05).sum()))
        bad = (err > 0.05).nonzero()
        print("   first bad", bad[:5].tolist())
        # try other experts' weights
        for e2 in range(E):
            p2 = X[e*seg:e*seg+c].float() @ W[e2].float().T + (bias[e] if use_bias else 0)
            print("     vs W", e2, float((got-p2).norm()/p2.norm()))
