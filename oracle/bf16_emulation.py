"""ORACLE / TEST INFRASTRUCTURE ONLY — numpy emulation of WHERE the B200 path
rounds to bf16 (dense block stack), used to separate the error inherent to the
bf16-in / fp32-accumulate design from kernel bugs. `points` selects which
tensors are rounded; an empty set reproduces p2r_oracle.Model exactly.
Mirrors Model::block_forward / block_backward in csrc/engine/engine.cpp.
"""
from __future__ import annotations

import numpy as np

from . import p2r_oracle as O

F32 = np.float32
ALL_POINTS = ("w16", "a16", "qkv16", "p16", "o16", "b16", "hpre16", "g16", "h16",
              "dlogits16", "dres16", "dh16", "dx1_16", "do16", "ds16", "dqkv16")


def bf16(x):
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def loss_and_grads(cfg: O.Config, params: dict, tokens, targets, mask, batch, denom, points=ALL_POINTS):
    pts = set(points)

    def R(x, tag):
        return bf16(x) if tag in pts else np.asarray(x, F32)

    P0 = {k: np.asarray(v, F32) for k, v in params.items()}
    W = {k: (R(v, "w16") if v.ndim >= 2 else v) for k, v in P0.items()}
    c = cfg
    T = len(tokens)
    S = T // batch
    H = c.n_heads
    d = c.d_model
    hd = d // H
    tok = np.asarray(tokens)
    pos = np.tile(np.arange(S), batch)
    x = (P0["embed.tok"][tok] + P0["embed.pos"][pos]).astype(F32)
    caches = []

    def pre(g):
        return "layer.0." if c.n_layers_params == 1 else f"layer.{g}."

    def attn_fwd(qkv):
        q, k, v = (O.split_heads(t, batch, H, S) for t in np.split(qkv, 3, axis=1))
        s = (q @ np.swapaxes(k, -1, -2)) * F32(1 / np.sqrt(hd))
        s = np.where(np.tril(np.ones((S, S), bool)), s, -np.inf)
        e = np.exp(s - s.max(-1, keepdims=True))
        l_ = e.sum(-1, keepdims=True)
        p = e / l_
        o = (R(e, "p16") @ v) / l_  # bf16(P) in the P.V MMA, fp32 normaliser
        return O.merge_heads(o.astype(F32)), (q, k, v, p)

    for g in range(c.n_layers_graph):
        pr = pre(g)
        a, xh1, inv1 = O.layernorm_fwd(x, P0[pr + "ln1.gain"], P0[pr + "ln1.bias"])
        a16 = R(a, "a16")
        wqkv = np.concatenate([W[pr + "attn.wq"], W[pr + "attn.wk"], W[pr + "attn.wv"]], 1)
        qkv = R(a16 @ wqkv, "qkv16")
        o, ac = attn_fwd(qkv)
        o16 = R(o, "o16")
        x1 = (x + o16 @ W[pr + "attn.wo"]).astype(F32)
        b, xh2, inv2 = O.layernorm_fwd(x1, P0[pr + "ln2.gain"], P0[pr + "ln2.bias"])
        b16 = R(b, "b16")
        hpre = (b16 @ W[pr + "ffn.w1"] + P0[pr + "ffn.b1"]).astype(F32)
        g16 = R(O.gelu_fwd(hpre), "g16")
        hpre16 = R(hpre, "hpre16")
        xn = (x1 + g16 @ W[pr + "ffn.w2"] + P0[pr + "ffn.b2"]).astype(F32)
        caches.append((x, a16, xh1, inv1, qkv, ac, o16, x1, b16, xh2, inv2, hpre16, g16, wqkv))
        x = xn
    h, xhf, invf = O.layernorm_fwd(x, P0["final_norm.gain"], P0["final_norm.bias"])
    h16 = R(h, "h16")
    logits = (h16 @ W["embed.tok"].T).astype(F32)
    loss, gl = O.cross_entropy_fwd_bwd(logits, targets, mask, denom)
    gl16 = R(gl, "dlogits16")
    G = {k: np.zeros_like(v) for k, v in P0.items()}
    G["embed.tok"] += gl16.T @ h16
    dh = gl16 @ W["embed.tok"]
    dres, gg, gb = O.layernorm_bwd(dh.astype(F32), xhf, invf, P0["final_norm.gain"])
    G["final_norm.gain"] += gg
    G["final_norm.bias"] += gb
    for g in reversed(range(c.n_layers_graph)):
        pr = pre(g)
        x, a16, xh1, inv1, qkv, (q, k, v, p), o16, x1, b16, xh2, inv2, hpre16, g16, wqkv = caches[g]
        dy = dres
        dy16 = R(dy, "dres16")
        G[pr + "ffn.w2"] += g16.T @ dy16
        G[pr + "ffn.b2"] += dy.sum(0)
        dh16 = R(O.gelu_bwd(dy16 @ W[pr + "ffn.w2"].T, hpre16), "dh16")
        G[pr + "ffn.w1"] += b16.T @ dh16
        G[pr + "ffn.b1"] += dh16.sum(0)
        db = (dh16 @ W[pr + "ffn.w1"].T).astype(F32)
        gx1, gg, gb = O.layernorm_bwd(db, xh2, inv2, P0[pr + "ln2.gain"])
        G[pr + "ln2.gain"] += gg
        G[pr + "ln2.bias"] += gb
        dx1 = (gx1 + dy).astype(F32)
        dx1_16 = R(dx1, "dx1_16")
        G[pr + "attn.wo"] += o16.T @ dx1_16
        do16 = R(dx1_16 @ W[pr + "attn.wo"].T, "do16")
        go = O.split_heads(do16, batch, H, S)
        scale = F32(1 / np.sqrt(hd))
        dP = go @ np.swapaxes(v, -1, -2)
        D = (go * O.split_heads(o16, batch, H, S)).sum(-1, keepdims=True)
        ds = R(p * (dP - D), "ds16")
        gq = scale * (ds @ k)
        gk = scale * (np.swapaxes(ds, -1, -2) @ q)
        gv = np.swapaxes(R(p, "p16"), -1, -2) @ go
        dqkv = R(np.concatenate([O.merge_heads(t) for t in (gq, gk, gv)], 1), "dqkv16")
        dw = a16.T @ dqkv
        G[pr + "attn.wq"] += dw[:, :d]
        G[pr + "attn.wk"] += dw[:, d:2 * d]
        G[pr + "attn.wv"] += dw[:, 2 * d:]
        da = (dqkv @ wqkv.T).astype(F32)
        gxa, gg, gb = O.layernorm_bwd(da, xh1, inv1, P0[pr + "ln1.gain"])
        G[pr + "ln1.gain"] += gg
        G[pr + "ln1.bias"] += gb
        dres = (gxa + dx1).astype(F32)
    np.add.at(G["embed.tok"], tok, dres)
    np.add.at(G["embed.pos"], pos, dres)
    return float(loss), G
