"""Granular CPU offload on the B200: a Real model with some layers kept in pinned
host DRAM (streamed through HBM staging slots, fused GPU AdamW in the backward)
trains BIT-IDENTICALLY to the same model fully resident, and moves exactly the
bytes its phase accounting says."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REAL_MOE = dict(d_model=256, d_ff=1024, n_layers_graph=4, n_layers_params=4, n_heads=4, vocab_size=260,
                seq_len=128, n_experts=4, n_prototypes=1)
REAL_DENSE = dict(d_model=256, d_ff=1024, n_layers_graph=5, n_layers_params=5, n_heads=4, vocab_size=260,
                  seq_len=128)


def lm_batch(batch, seq, seed=7):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


@pytest.mark.parametrize("cfgd,plan,ring", [(REAL_MOE, [1, 0, 1, 1], 2), (REAL_DENSE, [1, 1, 0, 1, 0], 3),
                                            (REAL_DENSE, [1, 1, 1, 1, 1], 2)],
                         ids=["moe_mixed_ring2", "dense_mixed_ring3", "dense_all_slow"])
@pytest.mark.parametrize("fn_form", ["master", "shadow"])
def test_offload_bit_identical_training(cuda, cfgd, plan, ring, fn_form, monkeypatch):
    """fn_form: the forward loads the fp32 master (default) or the bf16 shadow
    (P2R_OFFLOAD_FN_SHADOW=1, read when the offloaded model is created)."""
    monkeypatch.setenv("P2R_OFFLOAD_FN_SHADOW", "1" if fn_form == "shadow" else "0")
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**cfgd)
    a = p2r.Model(cfg, 1234)
    b = p2r.Model(cfg, 1234, offload=plan, ring_slots=ring)
    pa, pb = a.params(), b.params()
    for n in pa:
        assert np.array_equal(pa[n], pb[n]), n
    a.attach_adamw()
    b.attach_adamw()
    # HBM holds the FAST granules + `ring` staging slots instead of every granule
    assert b.device_param_bytes() < a.device_param_bytes() or ring >= sum(plan)
    b.offload_stats_reset()
    for s in range(3):
        tok, tgt, mask = lm_batch(4, 128, seed=10 + s)
        lr = 1e-3 * (s + 1)
        b.set_offload_lr(lr)
        la = a.train_step(tok, tgt, mask, 4, float(mask.sum()))
        lb = b.train_step(tok, tgt, mask, 4, float(mask.sum()))
        assert la == lb, (s, la, lb)
        a.adamw_step(lr)
        b.adamw_step(lr)
    pa, pb = a.params(), b.params()
    ma, mb = a.moments(), b.moments()
    for n in pa:
        assert np.array_equal(pa[n], pb[n]), n
        assert np.array_equal(ma[n][0], mb[n][0]) and np.array_equal(ma[n][1], mb[n][1]), n
    # phase accounting per SLOW granule per step: Fn = bf16 shadow (2 B/elem) + the
    # fp32 vectors / gate the forward reads, or the fp32 master (4); Bn = fp32 master (4);
    # moments 8; write-back p, m, v (12) + the bf16 shadow (2) in the shadow form
    st = b.offload_stats()
    tok, _, _ = lm_batch(2, 128, seed=99)
    assert np.array_equal(a.forward(tok, 2), b.forward(tok, 2))
    g = b.layer_granule_bytes() // 18  # elements per granule (padded)
    ns = sum(plan)
    d, dff, E = cfgd["d_model"], cfgd["d_ff"], cfgd.get("n_experts", 0)
    fp32_elems = 4 * d + (d * E + E * dff + E * d if E else dff + d)
    shadow = fn_form == "shadow"
    assert st["Fn_load"] == 3 * ns * ((g * 2 + fp32_elems * 4) if shadow else g * 4)
    assert st["Bn_load"] == 3 * ns * g * 4
    assert st["opt_load"] == 3 * ns * g * 8
    assert st["writeback"] == 3 * ns * g * (14 if shadow else 12)
    assert st["h2d_ms"] > 0 and st["d2h_ms"] > 0


def test_offload_gradient_offload_without_optimizer(cuda):
    """No optimizer attached: SLOW-granule gradients are offloaded to host (SPEC's grad phase)."""
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**REAL_DENSE)
    plan = [0, 1, 0, 1, 1]
    a = p2r.Model(cfg, 1234)
    b = p2r.Model(cfg, 1234, offload=plan)
    tok, tgt, mask = lm_batch(4, 128)
    assert a.train_step(tok, tgt, mask, 4, float(mask.sum())) == b.train_step(tok, tgt, mask, 4, float(mask.sum()))
    ga, gb = a.grads(), b.grads()
    for n in ga:
        assert np.array_equal(ga[n], gb[n]), n
    st = b.offload_stats()
    assert st["grad_offload"] == sum(plan) * (b.layer_granule_bytes() // 18) * 4
