"""Print the per-iteration clock64 timeline of the heaviest dQ CTA (B=1, causal).

Needs the trace build: python scripts/attn_variants.py trace, then
P2R_LIB=build/exp/libp2r_trace.so python scripts/attn_trace.py
"""
import ctypes
import sys
import torch
sys.path.insert(0, ".")
from paper_2110_03888_b200 import _lib

L = _lib.lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
B, H, S, hd = (8 if ("--kv" in sys.argv or "--fwd8" in sys.argv or "--pp8" in sys.argv) else 1), 16, 1024, 64
d = H * hd
qkv = (torch.randn(B * S, 3 * d, device="cuda") * 0.5).bfloat16()
o = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * H * S, device="cuda")
do = torch.randn(B * S, d, device="cuda").bfloat16()
dsum = torch.empty(B * H * S, device="cuda")
dqkv = torch.empty(B * S, 3 * d, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _lib.check(L.p2r_attention_fwd(P(qkv), P(o), P(lse), B, H, S, d, 1, st))
    _lib.check(L.p2r_attention_bwd(P(qkv), P(o), P(lse), P(do), P(dsum), P(dqkv), B, H, S, d, 1, st))
torch.cuda.synchronize()
t = o.view(torch.int64).flatten()[:512].cpu().numpy() if "--fwd" not in sys.argv else None
t0 = None if t is None else (t[0] if not ("--pp" in sys.argv or "--pp8" in sys.argv) else min(v for v in t[16:300] if v > 0))
rel = lambda v: int(v - t0)
if "--fwd" in sys.argv or "--fwd8" in sys.argv:
    t = lse.view(torch.int64).flatten()[:256].cpu().numpy()
    t0 = t[0]
    print("fwd CTA (last q tile): setup->end", t[1] - t0)
    print(" j | mma: kvfull  S-issued  p_full(j) PV-issued | sm(warp4): sfull  max-done  exps-done  arrived")
    for j in range(22):
        m = [t[8 + 4 * j + i] for i in range(4)]
        a = [t[100 + 4 * j + i] for i in range(4)]
        f = lambda v: f"{v - t0:8d}" if 0 < v - t0 < 10**9 else "       -"
        print(f"{j:2d} | " + " ".join(f(v) for v in m) + " | " + " ".join(f(v) for v in a))
    sys.exit(0)
if "--kv" in sys.argv:  # dK/dV kernel, CTA 0 (B=8 shape: persistent items)
    t = o.view(torch.int64).flatten()[512:1024].cpu().numpy()
    v = [x for x in t if x > 0]
    t0 = min(v)
    g = lambda i: f"{t[i] - t0:8d}" if t[i] > 0 else "       -"
    print(" blk | mma1: qfull S(X0) S(X1) | dVdK done X0 X1 | X0: sfull arrive | X1: sfull arrive")
    for j in range(24):
        print(f"{j:4d} | {g(16 + 4 * j)} {g(17 + 4 * j)} {g(18 + 4 * j)} | {g(120 + j)} {g(168 + j)} | "
              f"{g(240 + 2 * j)} {g(241 + 2 * j)} | {g(368 + 2 * j)} {g(369 + 2 * j)}")
    sys.exit(0)
if "--pp" in sys.argv or "--pp8" in sys.argv:
    print(" j | mma: kvfull(j+1) S(j+1)issued dQA(j) dQB(j) | A: sfull  sfree  stored  dsfull | B: sfull  sfree  stored  dsfull")
    for j in range(16):
        m = [t[16 + 4 * j + i] for i in range(4)]
        a = [t[100 + 4 * j + i] for i in range(4)]
        b = [t[300 + 4 * j + i] for i in range(4)]  # group B: trb = 100 + 200
        f = lambda v: f"{rel(v):8d}" if 0 < v - t0 < 10**9 else "       -"
        print(f"{j:2d} | " + " ".join(f(v) for v in m) + " | " + " ".join(f(v) for v in a) + " | " + " ".join(f(v) for v in b))
    sys.exit(0)
print("after setup sync", rel(t[1]), " q_full (mma)", rel(t[2]), " D done (softmax)", rel(t[3]), " end", rel(t[4]))
print(" j | mma: kv_full  S-issued  ds_full(j) dQ-issued | sm: s_full  tmem_ld  math  dq_done  stored  arrived")
for j in range(16):
    m = t[16 + 4 * j:16 + 4 * j + 4]
    s = t[100 + 6 * j:100 + 6 * j + 6]
    print(f"{j:2d} | " + " ".join(f"{rel(v):8d}" for v in m) + " | " + " ".join(f"{rel(v):8d}" for v in s))
