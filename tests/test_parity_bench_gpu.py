"""Step parity at the configurations the benchmark and the north star run
(VERDICT r1 "next" #1), against the compiled reference (oracle/_ref):

* C2 bench config: d=1024, 16 heads, d_ff=4096, 24 graph layers sharing ONE
  parameter layer, seq 1024 (B=1 so the single-threaded reference finishes
  in ~20 s);
* C3 width: Real (delinked, unshared) MoE, d=1024, 8 experts top-1;
* SPEC acceptance #4: the Pseudo model's shared gradient
  equals the sum of the delinked clones' per-layer gradients (<= 1e-5);
* routing flips at E=64 with their logit gaps.

Tolerances (north star, tests/_parity.py): loss <= 1e-3 relative; every
parameter gradient <= 1e-2 relative L2, or <= 1.25x the bf16-in design's own
floor on the same inputs where that floor is already ~1e-2. That happens for
the attention Q/K projection gradients at random init: a tiny, ill-conditioned
signal (near-uniform attention, dQ ~ dO^T Cov(v, k)) that bf16 inputs put at
~0.8-1.4 % from the fp32 reference no matter which single rounding point is
raised to fp32 (oracle/precision_floor.py, profiles/r02_precision_floor.txt:
dropping the dQ/dK -> dW_qkv rounding moves the worst tensor 1.37 % -> 1.36 %;
the error is spread over every forward rounding point, weights included)."""
import os

import numpy as np
import pytest

from oracle import p2r_oracle as O

pytestmark = pytest.mark.gpu
REF_SO = os.path.join(os.path.dirname(__file__), "..", "oracle", "_ref", "libp2r_ref.so")
need_ref = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")

C2 = dict(d_model=1024, d_ff=4096, n_layers_graph=24, n_layers_params=1, n_heads=16, vocab_size=260,
          seq_len=1024)
C3W = dict(d_model=1024, d_ff=4096, n_layers_graph=2, n_layers_params=2, n_heads=16, vocab_size=260,
           seq_len=1024, n_experts=8, n_prototypes=1)


def lm_batch(batch, seq, seed=7):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


from ._parity import check_grads, design_floor, rel


@need_ref
def test_c2_bench_config_step_parity(cuda):
    """The benchmarked workload itself (bench.py C2) at B=1: loss and every gradient."""
    from oracle import ref
    import paper_2110_03888_b200 as p2r
    B, S = 1, C2["seq_len"]
    m = p2r.Model(p2r.Config(**C2), 1234)
    r = ref.RefModel(ref.Config(**C2), 1234)
    tok, tgt, mask = lm_batch(B, S)
    denom = float(mask.sum())
    lg = m.train_step(tok, tgt, mask, B, denom)
    p0 = r.params()
    lr_ = r.train_step(tok, tgt, mask, B, denom)
    print(f"C2 loss gpu {lg:.7f} ref {lr_:.7f} rel {abs(lg - lr_) / abs(lr_):.2e}")
    assert abs(lg - lr_) <= 1e-3 * abs(lr_)
    ge = design_floor(C2, p0, tok, tgt, mask, B, denom)
    check_grads(m.grads(), r.grads(), ge, r.names, "C2", strict=False)  # 24 layers: Q/K at the design floor


@need_ref
def test_c3_width_real_moe_parity(cuda):
    """Delinked (Real) MoE at the C3 width: d=1024, 8 experts top-1, two layers.
    Loss vs the compiled reference; gradients vs the oracle restatement under
    the GPU's routing (a flip moves whole tokens between experts), flips vs the
    oracle's own fp32 routing logged with their fp32 logit gap."""
    from oracle import ref
    import paper_2110_03888_b200 as p2r
    B, S = 1, C3W["seq_len"]
    T = B * S
    m = p2r.Model(p2r.Config(**C3W), 1234)
    r = ref.RefModel(ref.Config(**C3W), 1234)
    tok, tgt, mask = lm_batch(B, S, seed=11)
    denom = float(mask.sum())
    p0 = r.params()
    lg = m.train_step(tok, tgt, mask, B, denom)
    lr_ = r.train_step(tok, tgt, mask, B, denom)
    print(f"C3-width loss gpu {lg:.7f} ref {lr_:.7f}")
    assert abs(lg - lr_) <= 1e-3 * abs(lr_)
    free = O.Model(O.Config(**C3W), p0)
    free.forward(tok, B, keep=True)
    forced, cascaded = {}, 0
    for g in range(C3W["n_layers_graph"]):
        sel, sur, raw, cap, drop = m.layer_routing(g, T)
        forced[g] = sel
        osel = free._cache[2][g][12][2].selected
        ol = free._cache[2][g][12][1]
        for t in np.nonzero(sel != osel)[0]:
            cascaded += 1
            print(f"free-run flip layer {g} token {t}: gpu {sel[t]} oracle {osel[t]} fp32 gap "
                  f"{ol[t, osel[t]] - ol[t, sel[t]]:.3e}")
    om = O.Model(O.Config(**C3W), p0)
    om.forced_selected = forced
    lo, go = om.loss_and_grads(tok, tgt, mask, B, denom)
    assert abs(lg - lo) <= 1e-3 * abs(lo)
    # routing parity proper: layer g's choice against the oracle's own choice on the
    # same earlier-layer routing (a free-running oracle also counts cascades: one early
    # flip changes every later token's attention input). Each flip is a near-tie.
    flips, worst = 0, 0.0
    for g in range(C3W["n_layers_graph"]):
        ol = om._cache[2][g][12][1]
        own = O.moe_dispatch_vectorized(ol, C3W["n_experts"], C3W["n_prototypes"], 1.25).selected
        for t in np.nonzero(forced[g] != own)[0]:
            flips += 1
            gap = float(ol[t, own[t]] - ol[t, forced[g][t]])
            worst = max(worst, gap / float(ol.std()))
            print(f"flip layer {g} token {t}: gpu {forced[g][t]} oracle {own[t]} fp32 gap {gap:.3e}")
    print(f"C3-width flips {flips} (free-run incl. cascades {cascaded}), worst gap / logit std {worst:.2e}")
    assert flips <= 0.005 * T * C3W["n_layers_graph"], flips
    assert worst <= 0.02, worst
    ge = design_floor(C3W, p0, tok, tgt, mask, B, denom, forced)
    check_grads(m.grads(), go, ge, r.names, "C3W")


@pytest.mark.parametrize("moe", [False, True], ids=["dense", "moe"])
def test_spec4_shared_grad_equals_clone_sum(cuda, moe):
    """SPEC acceptance #4: L=3 shared-layer gradient == sum of the
    unshared clones' gradients (<= 1e-5 rel-L2) on the GPU path. The delinked model
    runs bitwise the same forward, so this checks the in-place (beta = 1) cross-layer
    accumulation of the dW epilogues against explicit per-layer gradients."""
    import paper_2110_03888_b200 as p2r
    cfgd = dict(d_model=256, d_ff=1024, n_layers_graph=3, n_layers_params=1, n_heads=4, vocab_size=260,
                seq_len=128)
    if moe:
        cfgd.update(n_experts=4, n_prototypes=1)
    m = p2r.Model(p2r.Config(**cfgd), 1234)
    real = m.delinked()
    tok, tgt, mask = lm_batch(4, 128, seed=3)
    denom = float(mask.sum())
    a = m.train_step(tok, tgt, mask, 4, denom)
    b = real.train_step(tok, tgt, mask, 4, denom)
    assert a == b  # bitwise-identical forward
    gs, gr = m.grads(), real.grads()
    worst = 0.0
    for n, v in gs.items():
        if not n.startswith("layer."):
            assert rel(v, gr[n]) <= 1e-5, n
            continue
        rest = n.split(".", 2)[2]
        acc = np.zeros_like(v)
        for i in reversed(range(3)):  # flush order of the reference (model.cpp:210-221)
            acc = (acc + gr[f"layer.{i}.{rest}"]).astype(np.float32)
        if np.linalg.norm(acc) == 0:
            assert np.abs(v).max() == 0.0, n
            continue
        e = rel(v, acc)
        worst = max(worst, e)
        assert e <= 1e-5, (n, e)
    print(f"shared grad vs sum of clone grads: worst rel-L2 {worst:.2e}")
    # sharing arithmetic: the Pseudo model holds ONE layer's gradient
    # granule (accumulated in place: no scratch set, so <= the reference's 2 layers), the
    # delinked model L of them; the embeddings granule is common to both
    cnt = p2r.count_params(p2r.Config(**cfgd))
    assert m.scratch_grad_bytes() == 0
    g1, g3 = m.grad_bytes(), real.grad_bytes()
    per_layer = (g3 - g1) // 2
    assert g3 == g1 + 2 * per_layer
    emb_params, layer_params, _ = cnt
    assert 4 * layer_params <= per_layer <= 4 * layer_params * 1.01  # (256-B aligned segments)
    assert 4 * emb_params <= g1 - per_layer <= 4 * emb_params * 1.01


@need_ref
def test_routing_flips_e64_logit_gaps(cuda):
    """E=64 (C4's expert count) end to end: every GPU-vs-fp32-oracle routing flip is
    listed with its fp32 logit gap, with the perturbation of the two logits that
    explains it; the GPU's gate logits stay within 1 % (rms) / 3 % (max) of the logit
    spread of the fp32 oracle's (fed the same upstream routing), and the flip rate
    stays below 1 %."""
    import paper_2110_03888_b200 as p2r
    cfgd = dict(d_model=1024, d_ff=512, n_layers_graph=2, n_layers_params=2, n_heads=16, vocab_size=260,
                seq_len=1024, n_experts=64, n_prototypes=1)
    B, S = 2, 1024
    T = B * S
    m = p2r.Model(p2r.Config(**cfgd), 1234)
    tok, tgt, mask = lm_batch(B, S, seed=5)
    m.train_step(tok, tgt, mask, B, float(mask.sum()))
    om = O.Model(O.Config(**cfgd), m.params())
    om.forced_selected = {}
    flips, gaps = 0, []
    for g in range(cfgd["n_layers_graph"]):
        sel, sur, raw, cap, drop = m.layer_routing(g, T)
        gl = m.gate_logits(g, T)
        om.forced_selected = {gg: m.layer_routing(gg, T)[0] for gg in range(g)}  # upstream layers as on the GPU
        om.forward(tok, B, keep=True)
        ol = om._cache[2][g][12][1]
        osel = O.moe_dispatch_vectorized(ol, 64, 1, 1.25).selected
        dl = np.abs(gl - ol)
        print(f"layer {g}: gate logit |gpu - fp32| max {dl.max():.3e} rms {np.sqrt((dl ** 2).mean()):.3e}")
        for t in np.nonzero(sel != osel)[0]:
            a, b = int(osel[t]), int(sel[t])
            gap = float(ol[t, a] - ol[t, b])
            expl = float(dl[t, a] + dl[t, b])
            print(f"  flip token {t}: gpu {b} fp32 {a}  fp32 gap {gap:.3e}  perturbation {expl:.3e}")
            gaps.append(gap)
            flips += 1
        # a flip needs fp32 gap <= the perturbation of the two logits, so bound the
        # perturbation itself against the spread of the logits (bf16-in upstream)
        assert np.sqrt((dl ** 2).mean()) <= 0.01 * float(ol.std()) and dl.max() <= 0.03 * float(ol.std()), \
            (dl.max(), ol.std())
    print(f"flips {flips} / {T * cfgd['n_layers_graph']}; max gap {max(gaps) if gaps else 0:.3e}")
    assert flips <= 0.01 * T * cfgd["n_layers_graph"]
