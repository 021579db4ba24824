"""The primitive layer behind the drop-in tensor API (csrc/prims.cu) against
numpy restatements of the reference primitives (tensor.cpp:131-723), through
the C-ABI on device buffers: generic shapes, fp32, deterministic order."""
import math

import numpy as np
import pytest

from ._gpu import call, dev

pytestmark = pytest.mark.gpu
F = np.float32


def host(t):
    return t.cpu().numpy()


def test_prim_gemm_all_layouts(cuda):
    import torch
    rng = np.random.default_rng(0)
    for (m, n, k) in [(1, 1, 2), (3, 5, 8), (17, 33, 19), (64, 48, 80)]:
        for ta in (0, 1):
            for tb in (0, 1):
                A = rng.standard_normal((k, m) if ta else (m, k)).astype(F)
                B = rng.standard_normal((n, k) if tb else (k, n)).astype(F)
                C = rng.standard_normal((m, n)).astype(F)
                want = (A.T if ta else A) @ (B.T if tb else B) + 0.5 * C
                dc = dev(C)
                call("prim_gemm_f32", ta, tb, m, n, k, dev(A), m if ta else k, dev(B), k if tb else n, dc, n,
                     0.5, 1, 0, 0, 0)
                assert np.allclose(host(dc), want, rtol=1e-5, atol=1e-5), (m, n, k, ta, tb)


def test_prim_elementwise_and_bias(cuda):
    import torch
    from oracle import p2r_oracle as O
    rng = np.random.default_rng(1)
    a = rng.standard_normal(1000).astype(F)
    b = rng.standard_normal(1000).astype(F)
    out = dev(np.zeros(1000, F))
    call("prim_ew", 0, 1000, dev(a), dev(b), out)
    assert np.array_equal(host(out), a + b)
    out = dev(np.zeros(1000, F))
    call("prim_ew", 2, 1000, dev(a), None, out)
    assert np.allclose(host(out), O.gelu_fwd(a), atol=2e-6)
    out = dev(np.ones(1000, F))
    call("prim_ew", 3, 1000, dev(a), dev(b), out)
    assert np.allclose(host(out), 1 + O.gelu_bwd(b, a), atol=2e-6)
    x = rng.standard_normal((7, 5)).astype(F)
    bias = rng.standard_normal(5).astype(F)
    out = dev(np.zeros((7, 5), F))
    call("prim_bias", 7, 5, dev(x), dev(bias), out)
    assert np.array_equal(host(out), x + bias)
    acc = dev(np.ones(5, F))
    call("prim_colsum_acc", 7, 5, dev(x), acc)
    assert np.allclose(host(acc), 1 + x.sum(0), atol=1e-5)


@pytest.mark.parametrize("d", [2, 5, 256, 300])
def test_prim_layernorm(cuda, d):
    from oracle import p2r_oracle as O
    rng = np.random.default_rng(2)
    x = rng.standard_normal((9, d)).astype(F)
    g = rng.standard_normal(d).astype(F)
    b = rng.standard_normal(d).astype(F)
    y, xh, iv = (dev(np.zeros(s, F)) for s in ((9, d), (9, d), 9))
    call("prim_layernorm_fwd", 9, d, dev(x), dev(g), dev(b), 1e-5, y, xh, iv)
    wy, wxh, winv = O.layernorm_fwd(x, g, b)
    assert np.allclose(host(y), wy, atol=1e-5) and np.allclose(host(iv), winv, rtol=1e-5)
    gy = rng.standard_normal((9, d)).astype(F)
    gx, gg, gb = dev(np.zeros((9, d), F)), dev(np.zeros(d, F)), dev(np.zeros(d, F))
    call("prim_layernorm_bwd", 9, d, dev(gy), xh, iv, dev(g), gx, gg, gb)
    wgx, wgg, wgb = O.layernorm_bwd(gy, wxh, winv, g)
    assert np.allclose(host(gx), wgx, atol=1e-4) and np.allclose(host(gg), wgg, atol=1e-4)
    assert np.allclose(host(gb), wgb, atol=1e-4)


def test_prim_rows_heads_softmax(cuda):
    from oracle import p2r_oracle as O
    rng = np.random.default_rng(3)
    x = rng.standard_normal((10, 6)).astype(F)
    rows = np.array([3, 0, 3, 9, 1], np.int32)
    out = dev(np.zeros((5, 6), F))
    call("prim_gather_rows", 5, 6, dev(x), dev(rows), out)
    assert np.array_equal(host(out), x[rows])
    g = rng.standard_normal((5, 6)).astype(F)
    gx = dev(np.zeros((10, 6), F))
    call("prim_scatter_rows_acc", 5, 6, dev(g), dev(rows), gx)
    want = np.zeros((10, 6), F)
    np.add.at(want, rows, g)
    assert np.allclose(host(gx), want, atol=1e-6)
    B, H, S, hd = 2, 3, 4, 5
    y = rng.standard_normal((B * S, H * hd)).astype(F)
    sp = dev(np.zeros((B, H, S, hd), F))
    call("prim_permute_heads", 0, 0, B, H, S, hd, dev(y), sp)
    assert np.array_equal(host(sp), O.split_heads(y, B, H, S))
    back = dev(np.zeros_like(y))
    call("prim_permute_heads", 1, 0, B, H, S, hd, sp, back)
    assert np.array_equal(host(back), y)
    s = rng.standard_normal((B * H * S, S)).astype(F)
    p = dev(s.copy())
    call("prim_softmax_rows", B * H * S, S, S, p)
    s4 = s.reshape(B, H, S, S)
    e = np.where(np.tril(np.ones((S, S), bool)), s4, -np.inf)
    want = np.exp(e - e.max(-1, keepdims=True))
    want = (want / want.sum(-1, keepdims=True)).reshape(-1, S)
    assert np.allclose(host(p), want, atol=1e-6)
    dp = rng.standard_normal(want.shape).astype(F)
    ds = dev(np.zeros_like(want))
    call("prim_softmax_bwd_rows", B * H * S, S, p, dev(dp), ds)
    assert np.allclose(host(ds), want * (dp - (want * dp).sum(-1, keepdims=True)), atol=1e-5)


def test_prim_selected_softmax_combine_ce(cuda):
    from oracle import p2r_oracle as O
    rng = np.random.default_rng(4)
    T, E, k, d = 12, 6, 2, 8
    logits = rng.standard_normal((T, E)).astype(F)
    r = O.moe_dispatch(logits, E, k, 0.8)
    w = dev(np.zeros((T, k), F))
    call("prim_selected_softmax", 0, T, E, k, dev(logits), None, dev(r.selected), dev(r.survived), w)
    ww = O.selected_softmax_fwd(logits, r)
    assert np.allclose(host(w), ww, atol=1e-6)
    gw = rng.standard_normal((T, k)).astype(F)
    gl = dev(np.zeros((T, E), F))
    call("prim_selected_softmax", 1, T, E, k, w, dev(gw), dev(r.selected), dev(r.survived), gl)
    assert np.allclose(host(gl), O.selected_softmax_bwd(gw, ww, r, E), atol=1e-5)
    # combine: token contributions in (expert, row) order
    ys = [rng.standard_normal((len(r.expert_rows[e]), d)).astype(F) for e in range(E)]
    y = np.concatenate(ys)
    rtok = np.concatenate([r.expert_rows[e] for e in range(E)]).astype(np.int32)
    rslot = np.concatenate([r.expert_slots[e] for e in range(E)]).astype(np.int32)
    off = np.zeros(T + 1, np.int32)
    np.add.at(off, rtok + 1, 1)
    off = np.cumsum(off).astype(np.int32)
    order = np.argsort(rtok, kind="stable")
    out = dev(np.zeros((T, d), F))
    call("prim_combine_fwd", T, d, k, dev(off), dev(order.astype(np.int32)), dev(rslot[order]), dev(y), w, out)
    want = np.zeros((T, d), F)
    for i, t in enumerate(rtok):
        want[t] += ww[t, rslot[i]] * y[i]
    assert np.allclose(host(out), want, atol=1e-5)
    dout = rng.standard_normal((T, d)).astype(F)
    dy, dw = dev(np.zeros_like(y)), dev(np.zeros((T, k), F))
    call("prim_combine_bwd", len(rtok), d, k, dev(rtok), dev(rslot), dev(dout), dev(y), w, dy, dw)
    assert np.allclose(host(dy), ww[rtok, rslot][:, None] * dout[rtok], atol=1e-5)
    wdw = np.zeros((T, k), F)
    for i, t in enumerate(rtok):
        wdw[t, rslot[i]] += (dout[t] * y[i]).sum()
    assert np.allclose(host(dw), wdw, atol=1e-4)
    V = 11
    lg = rng.standard_normal((T, V)).astype(F)
    tg = rng.integers(0, V, T).astype(np.int32)
    mask = (rng.random(T) > 0.2).astype(np.uint8)
    import torch
    ws = torch.zeros(T, dtype=torch.float64, device="cuda")
    loss, g = dev(np.zeros(1, F)), dev(np.zeros((T, V), F))
    call("prim_cross_entropy", T, V, dev(lg), dev(tg), dev(mask), __import__("ctypes").c_double(7.0), ws, loss, g)
    wl, wg = O.cross_entropy_fwd_bwd(lg, tg, mask, 7.0)
    assert abs(float(host(loss)[0]) - float(wl)) <= 1e-6 * abs(float(wl)) + 1e-7
    assert np.allclose(host(g), wg, atol=1e-6)
