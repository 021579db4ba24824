"""Diagnostic: attention fwd/bwd error vs fp64 on the SAME bf16 inputs, at
model-like scales (init weights 0.02) and unit scale."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
from tests._gpu import call, dev
from oracle import p2r_oracle as O

def bf(x): return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().float().numpy()
def run(scale_in, B=2, H=4, S=128, hd=64, causal=1):
    rng = np.random.default_rng(0)
    d = H*hd
    q, k, v = (bf(rng.standard_normal((B, H, S, hd)) * scale_in) for _ in range(3))
    go = bf(rng.standard_normal((B, H, S, hd)) * 1e-3)
    qkv = np.concatenate([O.merge_heads(q), O.merge_heads(k), O.merge_heads(v)], 1)
    QKV = dev(qkv, torch.bfloat16)
    o = torch.empty(B*S, d, dtype=torch.bfloat16, device="cuda"); lse = torch.empty(B*H*S, device="cuda")
    call("attention_fwd", QKV, o, lse, B, H, S, d, causal)
    # fp64 reference on the same inputs
    q64, k64, v64, go64 = (x.astype(np.float64) for x in (q, k, v, go))
    s = q64 @ np.swapaxes(k64, -1, -2) / 8
    if causal: s = np.where(np.tril(np.ones((S, S), bool)), s, -np.inf)
    p = np.exp(s - s.max(-1, keepdims=True)); p /= p.sum(-1, keepdims=True)
    O64 = p @ v64
    GO = dev(O.merge_heads(go), torch.bfloat16)
    dsum = torch.empty(B*H*S, device="cuda"); dqkv = torch.empty(B*S, 3*d, dtype=torch.bfloat16, device="cuda")
    call("attention_bwd", QKV, o, lse, GO, dsum, dqkv, B, H, S, d, causal)
    dP = go64 @ np.swapaxes(v64, -1, -2); D = (p*dP).sum(-1, keepdims=True); dS = p*(dP - D)
    gq = dS @ k64 / 8; gk = np.swapaxes(dS, -1, -2) @ q64 / 8; gv = np.swapaxes(p, -1, -2) @ go64
    out = dqkv.float().cpu().numpy()
    r = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    print(f"scale {scale_in}: O {r(o.float().cpu().numpy(), O.merge_heads(O64)):.2e}  dq {r(out[:, :d], O.merge_heads(gq)):.2e}  "
          f"dk {r(out[:, d:2*d], O.merge_heads(gk)):.2e}  dv {r(out[:, 2*d:], O.merge_heads(gv)):.2e}  "
          f"(bf16 rounding of exact: dq {r(bf(O.merge_heads(gq)), O.merge_heads(gq)):.2e})")
for sc in (0.3, 1.0, 3.0):
    run(sc)
