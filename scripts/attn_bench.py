"""Attention fwd/bwd timing (CUDA events) at the C2 shape; P2R_LIB=build/libp2r_diag.so P2R_ATTN_MMA_SYNC=1
selects the legacy mma.sync kernels of the diagnostic build."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
from paper_2110_03888_b200 import _lib

L = _lib.lib()
B, H, S, hd = 8, 16, 1024, 64
if len(sys.argv) > 1:
    hd = int(sys.argv[1])
    H = 1024 // hd
d = H * hd
qkv = (torch.randn(B * S, 3 * d, device="cuda") * 0.5).bfloat16()
o = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
do = torch.randn(B * S, d, device="cuda").bfloat16()
dsum = torch.empty(B * H * S, device="cuda")
dqkv = torch.empty(B * S, 3 * d, device="cuda", dtype=torch.bfloat16)
flops = 2.0 * B * H * S * S * hd  # causal fwd (QK^T + PV over the lower triangle)
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def fwd():
    _lib.check(L.p2r_attention_fwd(P(qkv), P(o), P(lse), B, H, S, d, 1, st))


def bwd():
    _lib.check(L.p2r_attention_bwd(P(qkv), P(o), P(lse), P(do), P(dsum), P(dqkv), B, H, S, d, 1, st))


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


f = t(fwd)
bw = t(bwd)
print(f"hd={hd}: attn fwd {f*1e3:.1f} us  {flops/f/1e9:.1f} TFLOP/s | bwd {bw*1e3:.1f} us  {2*flops/bw/1e9:.1f} TFLOP/s")
