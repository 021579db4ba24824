"""Attention fwd/bwd time vs batch (waves of CTAs) at S=1024, hd=64 (diagnostic)."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
from paper_2110_03888_b200 import _lib

L = _lib.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def bench(B, H=16, S=1024, hd=64, causal=1, it=20):
    d = H * hd
    qkv = (torch.randn(B * S, 3 * d, device="cuda") * 0.5).bfloat16()
    o = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * H * S, device="cuda")
    do = torch.randn(B * S, d, device="cuda").bfloat16()
    dsum = torch.empty(B * H * S, device="cuda")
    dqkv = torch.empty(B * S, 3 * d, device="cuda", dtype=torch.bfloat16)
    fwd = lambda: _lib.check(L.p2r_attention_fwd(P(qkv), P(o), P(lse), B, H, S, d, causal, st))
    bwd = lambda: _lib.check(L.p2r_attention_bwd(P(qkv), P(o), P(lse), P(do), P(dsum), P(dqkv), B, H, S, d, causal, st))
    res = []
    for fn in (fwd, bwd):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(it):
            fn()
        b.record()
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b) / it * 1e3)
    ctas = B * H * (S // 128)
    print(f"B={B:2d} H={H} S={S} causal={causal} CTAs/kernel={ctas:5d} waves={ctas/148:5.2f}: fwd {res[0]:7.1f} us  bwd {res[1]:7.1f} us")


for B in (1, 2, 4, 8):
    bench(B)
bench(1, H=9)
bench(8, causal=0)
