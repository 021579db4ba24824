"""LayerNorm fwd/bwd + column-sum kernel timings (CUDA events) at the C2 shape."""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
from paper_2110_03888_b200 import _lib

L = _lib.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
T, d = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (8192, 1024)
x = torch.randn(T, d, device="cuda")
g = torch.randn(d, device="cuda")
b = torch.randn(d, device="cuda")
y16 = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
mean = torch.empty(T, device="cuda")
rstd = torch.empty(T, device="cuda")
dy = torch.randn(T, d, device="cuda")
res = torch.randn(T, d, device="cuda")
dx = torch.empty(T, d, device="cuda")
dx16 = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
gg = torch.zeros(d, device="cuda")
gb = torch.zeros(d, device="cuda")
ws = torch.empty(L.p2r_layernorm_bwd_workspace(T, d) // 4 + 1, device="cuda")
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def t(fn, it=20, cold=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(it):
        if cold:
            flush.zero_()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(e)
    return tot / it * 1e3


fwd = lambda: _lib.check(L.p2r_layernorm_fwd(P(x), P(g), P(b), T, d, ctypes.c_float(1e-5), P(y16), None, P(mean), P(rstd), st))
bwd = lambda: _lib.check(L.p2r_layernorm_bwd(P(dy), P(x), P(mean), P(rstd), P(g), P(res), T, d, P(dx), P(dx16), P(gg), P(gb), P(ws), st))
def b2b(fn, it=20):
    """back-to-back launches (PDL overlaps launch latency, as inside the step)"""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    e.record()
    torch.cuda.synchronize()
    return a.elapsed_time(e) / it * 1e3


dy16 = dy.bfloat16()
bwd16 = lambda: _lib.check(L.p2r_layernorm_bwd_fused_bf16(P(dy16), P(x), P(mean), P(rstd), P(g), P(res), T, d, P(dx),
                                                         P(dx16), P(gg), P(gb), P(ws), None, None, 0, None, st))
b16 = b2b(bwd16)
print(f"T={T} d={d} back-to-back: ln bwd (bf16 dy, the step's form) {b16:6.1f} us ({(T*d*16)/b16/1e3:6.0f} GB/s)")
f, bw = b2b(fwd), b2b(bwd)
print(f"T={T} d={d} back-to-back: ln fwd {f:6.1f} us ({(T*d*6)/f/1e3:6.0f} GB/s)  ln bwd {bw:6.1f} us ({(T*d*18)/bw/1e3:6.0f} GB/s)")
for cold in (True, False):
    f, bw = t(fwd, cold=cold), t(bwd, cold=cold)
    print(f"T={T} d={d} {'cold' if cold else 'warm'}: ln fwd {f:6.1f} us ({(T*d*6)/f/1e3:6.0f} GB/s)  "
          f"ln bwd {bw:6.1f} us ({(T*d*18)/bw/1e3:6.0f} GB/s)")
