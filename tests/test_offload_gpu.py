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
    """fn_form: the forward loads the bf16 shadow + fp32 vectors (default) or the fp32
    master (P2R_OFFLOAD_FN_SHADOW=0, read when the offloaded model is created)."""
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
    # (the shadow form writes the fp32 vectors back ahead of the master, with the shadow)
    assert st["writeback"] == 3 * ns * (g * 14 + fp32_elems * 4 if shadow else g * 12)
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


@pytest.mark.parametrize("plan", [[1, 0, 1, 1, 0], [1, 1, 1, 1, 1]], ids=["mixed", "all_slow"])
def test_offload_accumulation_bit_identical(cuda, plan):
    """Gradient accumulation (zero=True, then zero=False micro-steps, SPEC.md:463 /
    tensor.hpp:135-140): SLOW granules park partial gradients in pinned host memory
    between micro-steps and take the fused AdamW in the window's LAST backward only,
    so two optimizer steps of 3 micro-steps each are bit-identical to the resident model."""
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**REAL_DENSE)
    a = p2r.Model(cfg, 1234)
    b = p2r.Model(cfg, 1234, offload=plan, ring_slots=2)
    a.attach_adamw()
    b.attach_adamw()
    b.set_grad_accumulation(3)
    b.offload_stats_reset()
    for step in range(2):
        lr = 1e-3 * (step + 1)
        b.set_offload_lr(lr)
        for micro in range(3):
            tok, tgt, mask = lm_batch(4, 128, seed=30 + 3 * step + micro)
            denom = float(mask.sum()) * 3  # large-batch mean over the window
            la = a.train_step(tok, tgt, mask, 4, denom, zero=(micro == 0))
            lb = b.train_step(tok, tgt, mask, 4, denom, zero=(micro == 0))
            assert la == lb, (step, micro)
            if micro == 1:  # partial gradients of SLOW granules are readable from the host park
                ga, gb = a.grads(), b.grads()
                for n in ga:
                    assert np.array_equal(ga[n], gb[n]), n
        a.adamw_step(lr)
        b.adamw_step(lr)
    pa, pb = a.params(), b.params()
    ma, mb = a.moments(), b.moments()
    for n in pa:
        assert np.array_equal(pa[n], pb[n]), n
        assert np.array_equal(ma[n][0], mb[n][0]) and np.array_equal(ma[n][1], mb[n][1]), n
    st = b.offload_stats()
    g = b.layer_granule_bytes() // 18
    ns = sum(plan)
    # per window: 2 parks (D2H) + 2 reloads (H2D) of the partial grads, moments once
    assert st["grad_offload"] == 2 * 2 * ns * g * 4
    assert st["grad_load"] == 2 * 2 * ns * g * 4
    assert st["opt_load"] == 2 * ns * g * 8


def test_offload_misuse_throws(cuda):
    """Offload misuse is loud: Pseudo models, a micro-step
    past the accumulation window, adamw_step before the window's last backward, a missing
    set_offload_lr, and a mismatched lr -- and a throwing adamw_step leaves the step count."""
    import paper_2110_03888_b200 as p2r
    with pytest.raises(p2r.P2RInvalidArgument, match="needs an unshared"):
        p2r.Model(p2r.Config(**dict(REAL_DENSE, n_layers_params=1)), 1, offload=[1])
    cfg = p2r.Config(**REAL_DENSE)
    b = p2r.Model(cfg, 1234, offload=[1, 0, 0, 0, 1])
    b.attach_adamw()
    tok, tgt, mask = lm_batch(2, 128)
    with pytest.raises(p2r.P2RLogicError, match="set_offload_lr"):
        b.train_step(tok, tgt, mask, 2, float(mask.sum()))
    b.set_offload_lr(1e-3)
    b.train_step(tok, tgt, mask, 2, float(mask.sum()))
    with pytest.raises(p2r.P2RLogicError, match="accumulation past the window"):
        b.train_step(tok, tgt, mask, 2, float(mask.sum()), zero=False)
    with pytest.raises(p2r.P2RLogicError, match="adamw_step\\(lr\\) was not called"):
        b.train_step(tok, tgt, mask, 2, float(mask.sum()))
    with pytest.raises(p2r.P2RInvalidArgument, match="pass the same lr"):
        b.adamw_step(2e-3)
    assert b.step_count() == 0
    b.adamw_step(1e-3)
    assert b.step_count() == 1
    b.set_grad_accumulation(2)
    b.train_step(tok, tgt, mask, 2, float(mask.sum()))
    with pytest.raises(p2r.P2RLogicError, match="before the accumulation window's last backward"):
        b.adamw_step(1e-3)
    assert b.step_count() == 1


@pytest.mark.parametrize("policy", [0, 1, 2], ids=["no_ckpt", "ckpt_slow", "ckpt_all"])
def test_offload_activation_checkpointing_bit_identical(cuda, policy):
    """Activation checkpointing: checkpointed layers keep only their output
    and recompute the rest in the backward -- same kernels, same operands, so the step
    is bit-identical to storing every activation (and to the resident model)."""
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**REAL_MOE)
    a = p2r.Model(cfg, 1234)
    b = p2r.Model(cfg, 1234, offload=[0, 1, 0, 1], ring_slots=2)
    b.set_activation_checkpointing(policy)
    a.attach_adamw()
    b.attach_adamw()
    for s in range(2):
        tok, tgt, mask = lm_batch(4, 128, seed=50 + s)
        b.set_offload_lr(1e-3)
        assert a.train_step(tok, tgt, mask, 4, float(mask.sum())) == b.train_step(tok, tgt, mask, 4,
                                                                                  float(mask.sum()))
        a.adamw_step(1e-3)
        b.adamw_step(1e-3)
    pa, pb = a.params(), b.params()
    for n in pa:
        assert np.array_equal(pa[n], pb[n]), n


def test_offload_with_expert_parallel_bit_identical(cuda, monkeypatch):
    """Offload + expert parallelism in one model (C5's shape of the engine): an EP shard
    (world 1, exchange path forced) with SLOW granules trains bit-identically to the
    resident EP shard."""
    monkeypatch.setenv("P2R_FORCE_EP", "1")
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**REAL_MOE)
    a = p2r.Model(cfg, 1234, ep=(1, 0))
    b = p2r.Model(cfg, 1234, offload=[1, 0, 1, 1], ring_slots=2, ep=(1, 0))
    uid = p2r.comm_unique_id()
    a.comm_init(uid)
    b.comm_init(p2r.comm_unique_id())
    a.attach_adamw()
    b.attach_adamw()
    for s in range(2):
        tok, tgt, mask = lm_batch(4, 128, seed=70 + s)
        b.set_offload_lr(1e-3)
        assert a.train_step(tok, tgt, mask, 4, float(mask.sum())) == b.train_step(tok, tgt, mask, 4,
                                                                                  float(mask.sum()))
        a.allreduce_grads()
        b.allreduce_grads()
        a.adamw_step(1e-3)
        b.adamw_step(1e-3)
    pa, pb = a.params(), b.params()
    for n in pa:
        assert np.array_equal(pa[n], pb[n]), n


def test_offload_pipelined_host_steps_bit_identical(cuda):
    """Model.train_step(wait=False) on an offloaded model (the SLOW granules' fused AdamW
    runs inside the backward, the write-back on the side streams): the next step is
    enqueued before the previous loss is read; losses, parameters and moments equal the
    resident model's synchronous loop bit for bit."""
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**REAL_MOE)
    a = p2r.Model(cfg, 1234)
    b = p2r.Model(cfg, 1234, offload=[1, 0, 1, 1], ring_slots=2)
    a.attach_adamw()
    b.attach_adamw()
    lr = 1e-3
    b.set_offload_lr(lr)
    batches = [lm_batch(4, 128, seed=30 + s) for s in range(4)]
    sync = []
    for tok, tgt, mask in batches:
        sync.append(a.train_step(tok, tgt, mask, 4, float(mask.sum())))
        a.adamw_step(lr)
    piped, prev = [], None
    for tok, tgt, mask in batches:
        cur = b.train_step(tok, tgt, mask, 4, float(mask.sum()), wait=False)
        b.adamw_step(lr)
        if prev is not None:
            piped.append(prev.value())
        prev = cur
    piped.append(prev.value())
    assert piped == sync
    pa, pb = a.params(), b.params()
    ma, mb = a.moments(), b.moments()
    for n in pa:
        assert np.array_equal(pa[n], pb[n]), n
        assert np.array_equal(ma[n][0], mb[n][0]) and np.array_equal(ma[n][1], mb[n][1]), n
