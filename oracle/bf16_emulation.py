"""ORACLE / TEST INFRASTRUCTURE ONLY — numpy emulation of WHERE the B200 path
rounds to bf16 (dense and MoE block stacks), used to separate the error inherent to the
bf16-in / fp32-accumulate design from kernel bugs. `points` selects which
tensors are rounded; an empty set reproduces p2r_oracle.Model exactly.
Mirrors Model::block_forward / block_backward in csrc/engine/engine.cpp.
"""
from __future__ import annotations

import numpy as np

from . import p2r_oracle as O

F32 = np.float32
ALL_POINTS = ("w16", "a16", "qkv16", "p16", "o16", "b16", "gd16", "g16", "h16",
              "dlogits16", "dres16", "dh16", "dx1_16", "do16", "ds16", "dqkv16", "ye16", "dye16", "dxe16",
              "dln16")


def bf16(x):
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def loss_and_grads(cfg: O.Config, params: dict, tokens, targets, mask, batch, denom, points=ALL_POINTS,
                   forced_selected=None, routing_out=None):
    """forced_selected: {graph layer: selected[T*k]} pins MoE routing (as the parity
    tests do with the GPU's routing); MoE layers without an entry route on their
    own (emulated) fp32 gate logits."""
    import math
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
        if c.moe:
            # fp32 gate on the fp32 LN2 output; experts read the bf16 rows (xe16 = b16)
            logits = (b @ P0[pr + "moe.gate"]).astype(F32)
            T_ = b.shape[0]
            if forced_selected is not None and g in forced_selected:
                cap = int(math.ceil(float(F32(c.capacity_factor)) * T_ / float(c.n_experts // c.n_prototypes)))
                rt = O.admit(forced_selected[g], c.n_experts, c.n_prototypes, cap)
            else:
                rt = O.moe_dispatch_vectorized(logits, c.n_experts, c.n_prototypes, c.capacity_factor)
            if routing_out is not None:
                routing_out[g] = rt.selected.copy()
            wgt = O.selected_softmax_fwd(logits, rt)
            y = np.zeros_like(b)
            ec = []
            for e in range(c.n_experts):
                rows = rt.expert_rows[e]
                if len(rows) == 0:
                    ec.append(None)
                    continue
                xe = b16[rows]
                he = (xe @ W[pr + f"moe.expert.{e}.w1"] + P0[pr + f"moe.expert.{e}.b1"]).astype(F32)
                ge16 = R(O.gelu_fwd(he), "g16")
                ye = R((ge16 @ W[pr + f"moe.expert.{e}.w2"] + P0[pr + f"moe.expert.{e}.b2"]).astype(F32), "ye16")
                wv = wgt[rows, rt.expert_slots[e]]
                y[rows] += wv[:, None] * ye
                # the forward epilogue stores gelu'(pre) in bf16 for the backward
                ec.append((xe, R(O.gelu_bwd(np.ones_like(he), he), "gd16"), ge16, ye))
            xn = (x1 + y).astype(F32)
            caches.append((x, a16, xh1, inv1, qkv, ac, o16, x1, b16, xh2, inv2, (b, logits, rt, wgt, ec), None, wqkv))
        else:
            hpre = (b16 @ W[pr + "ffn.w1"] + P0[pr + "ffn.b1"]).astype(F32)
            g16 = R(O.gelu_fwd(hpre), "g16")
            hpre16 = R(O.gelu_bwd(np.ones_like(hpre), hpre), "gd16")  # stored GELU derivative
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
    dres, gg, gb = O.layernorm_bwd(R(dh, "dln16"), xhf, invf, P0["final_norm.gain"])
    G["final_norm.gain"] += gg
    G["final_norm.bias"] += gb
    for g in reversed(range(c.n_layers_graph)):
        pr = pre(g)
        x, a16, xh1, inv1, qkv, (q, k, v, p), o16, x1, b16, xh2, inv2, hpre16, g16, wqkv = caches[g]
        dy = dres
        if c.moe:
            bm, logits, rt, wgt, ec = hpre16
            db = np.zeros_like(bm)
            gw = np.zeros_like(wgt)
            for e in reversed(range(c.n_experts)):
                if ec[e] is None:
                    continue
                xe, he16, ge16, ye = ec[e]
                rows, slots = rt.expert_rows[e], rt.expert_slots[e]
                wv = wgt[rows, slots]
                dye = R((wv[:, None] * dy[rows]).astype(F32), "dye16")
                gw[rows, slots] += (dy[rows] * ye).sum(-1, dtype=F32)
                G[pr + f"moe.expert.{e}.w2"] += ge16.T @ dye
                G[pr + f"moe.expert.{e}.b2"] += dye.sum(0)
                dhe = R((dye @ W[pr + f"moe.expert.{e}.w2"].T) * he16, "dh16")
                G[pr + f"moe.expert.{e}.w1"] += xe.T @ dhe
                G[pr + f"moe.expert.{e}.b1"] += dhe.sum(0)
                np.add.at(db, rows, R((dhe @ W[pr + f"moe.expert.{e}.w1"].T).astype(F32), "dxe16"))
            glog = O.selected_softmax_bwd(gw, wgt, rt, c.n_experts)
            G[pr + "moe.gate"] += (bm.T @ glog).astype(F32)
            db += (glog @ P0[pr + "moe.gate"].T).astype(F32)
        else:
            dy16 = R(dy, "dres16")
            G[pr + "ffn.w2"] += g16.T @ dy16
            G[pr + "ffn.b2"] += dy.sum(0)
            dh16 = R((dy16 @ W[pr + "ffn.w2"].T) * hpre16, "dh16")
            G[pr + "ffn.w1"] += b16.T @ dh16
            G[pr + "ffn.b1"] += dh16.sum(0)
            db = R((dh16 @ W[pr + "ffn.w1"].T).astype(F32), "dln16")
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
        da = R((dqkv @ wqkv.T).astype(F32), "dln16")
        gxa, gg, gb = O.layernorm_bwd(da, xh1, inv1, P0[pr + "ln1.gain"])
        G[pr + "ln1.gain"] += gg
        G[pr + "ln1.bias"] += gb
        dres = (gxa + dx1).astype(F32)
    np.add.at(G["embed.tok"], tok, dres)
    np.add.at(G["embed.pos"], pos, dres)
    return float(loss), G
