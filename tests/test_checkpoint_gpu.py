"""Checkpoint container + Pseudo->Real hand-off (SPEC.md:260-264,
:276-284, :307-308, :320), through the C-ABI.

Contracts checked bit-for-bit: save -> load -> train k steps == train k steps
uninterrupted; delink(pseudo checkpoint) gives a REAL checkpoint whose
logits equal the Pseudo model's and whose every layer carries the shared layer's
weights and AdamW moments."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C1 = dict(d_model=256, d_ff=1024, n_layers_graph=4, n_layers_params=1, n_heads=4, vocab_size=260,
          seq_len=128, n_experts=4, n_prototypes=1)
DENSE = dict(d_model=256, d_ff=1024, n_layers_graph=3, n_layers_params=1, n_heads=4, vocab_size=260,
             seq_len=128)
REAL = dict(d_model=256, d_ff=1024, n_layers_graph=3, n_layers_params=3, n_heads=4, vocab_size=260,
            seq_len=128)


def lm_batch(batch, seq, seed):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


def step(m, k, seed):
    tok, tgt, mask = lm_batch(8, 128, seed)
    loss = m.train_step(tok, tgt, mask, 8, float(mask.sum()))
    m.adamw_step(1e-3 * (1 + k))
    return loss


def assert_same_state(a, b):
    pa, pb = a.params(), b.params()
    ma, mb = a.moments(), b.moments()
    assert a.names == b.names
    for n in a.names:
        assert np.array_equal(pa[n], pb[n]), n
        assert np.array_equal(ma[n][0], mb[n][0]) and np.array_equal(ma[n][1], mb[n][1]), n
    assert a.step_count() == b.step_count()


@pytest.mark.parametrize("cfgd", [C1, DENSE, REAL], ids=["pseudo_moe", "pseudo_dense", "real"])
def test_resume_bit_identical(cuda, tmp_path, cfgd):
    """loading a checkpoint and continuing reproduces the run bit-for-bit."""
    import paper_2110_03888_b200 as p2r
    from paper_2110_03888_b200.checkpoint import read_buffer, read_manifest
    a = p2r.Model(p2r.Config(**cfgd), 1234)
    a.attach_adamw()
    for k in range(2):
        step(a, k, seed=100 + k)
    path = str(tmp_path / "mid.p2rckpt")
    a.save_checkpoint(path, global_step=2, samples_consumed=2 * 8 * 128, wall_time_s=1.5, rng_state=77,
                      last_eval_step=0)
    man = read_manifest(path)
    assert man["stage"] == ("PSEUDO" if p2r.Config(**cfgd).shared() else "REAL")
    assert man["config"]["d_model"] == cfgd["d_model"] and man["adamw"]["step_count"] == 2
    assert len(man["order"]) == 3 * len(a.names)
    # the host-side reader sees exactly the model's buffers
    pa = a.params()
    assert np.array_equal(read_buffer(path, "param/" + a.names[1], man), pa[a.names[1]])
    b, st = p2r.load_checkpoint(path)
    assert st == {"stage": man["stage"], "global_step": 2, "samples_consumed": 2048, "wall_time_s": 1.5,
                  "rng_state": 77, "last_eval_step": 0}
    assert_same_state(a, b)
    for k in range(2, 4):
        la, lb = step(a, k, seed=100 + k), step(b, k, seed=100 + k)
        assert la == lb
    assert_same_state(a, b)


def test_delink_checkpoint(cuda, tmp_path):
    """[OP] delink(pseudo_checkpoint) -> REAL checkpoint."""
    import paper_2110_03888_b200 as p2r
    m = p2r.Model(p2r.Config(**C1), 1234)
    m.attach_adamw()
    step(m, 0, seed=5)
    pseudo, real_path = str(tmp_path / "pseudo.p2rckpt"), str(tmp_path / "real.p2rckpt")
    m.save_checkpoint(pseudo, global_step=1)
    st = p2r.delink_checkpoint(pseudo, real_path)
    assert st["stage"] == "REAL" and st["global_step"] == 1
    r, st2 = p2r.load_checkpoint(real_path)
    assert st2["stage"] == "REAL" and r.cfg.n_layers_params == C1["n_layers_graph"]
    assert r.step_count() == m.step_count()
    tok, _, _ = lm_batch(8, 128, seed=6)
    assert np.array_equal(m.forward(tok, 8), r.forward(tok, 8))  # delink equivalence, bitwise
    pp, pr, mp, mr = m.params(), r.params(), m.moments(), r.moments()
    for n in pp:
        if not n.startswith("layer."):
            assert np.array_equal(pp[n], pr[n]), n
            continue
        rest = n.split(".", 2)[2]
        for i in range(C1["n_layers_graph"]):
            assert np.array_equal(pr[f"layer.{i}.{rest}"], pp[n]), n
            assert np.array_equal(mr[f"layer.{i}.{rest}"][0], mp[n][0])
            assert np.array_equal(mr[f"layer.{i}.{rest}"][1], mp[n][1])
    # the Real checkpoint cannot be delinked again; an inference-only model has no moments
    with pytest.raises(p2r.P2RLogicError, match="not in the PSEUDO stage"):
        p2r.delink_checkpoint(real_path, str(tmp_path / "again.p2rckpt"))


def test_checkpoint_errors(cuda, tmp_path):
    import paper_2110_03888_b200 as p2r
    m = p2r.Model(p2r.Config(**DENSE), 1)
    path = str(tmp_path / "d.p2rckpt")
    m.save_checkpoint(path)  # no optimizer attached: parameters only
    other = p2r.Model(p2r.Config(**{**DENSE, "d_ff": 512}), 1)
    with pytest.raises(p2r.P2RInvalidArgument, match="config does not match"):
        other.load_checkpoint(path)
    bad = str(tmp_path / "bad.p2rckpt")
    with open(path, "rb") as f:
        raw = bytearray(f.read())
    raw[0:8] = b"NOTACKPT"
    open(bad, "wb").write(bytes(raw))
    with pytest.raises(p2r.P2RError, match="not a p2r checkpoint"):
        m.load_checkpoint(bad)
    trunc = str(tmp_path / "trunc.p2rckpt")
    open(trunc, "wb").write(bytes(raw[:len(raw) // 2]).replace(b"NOTACKPT", b"P2RCKPT\x00", 1))
    with pytest.raises(p2r.P2RError, match="truncated"):
        m.load_checkpoint(trunc)
    # parameters-only checkpoint loads into a model and leaves its optimizer detached
    b, st = p2r.load_checkpoint(path)
    assert st["stage"] == "PSEUDO"
    pa, pb = m.params(), b.params()
    for n in m.names:
        assert np.array_equal(pa[n], pb[n])


def test_load_into_offloaded_model(cuda, tmp_path):
    """A REAL checkpoint loads into a model whose layers live in pinned host memory
    (granular offload) and trains identically to the resident model."""
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**REAL)
    a = p2r.Model(cfg, 7)
    a.attach_adamw()
    step(a, 0, seed=11)
    path = str(tmp_path / "real.p2rckpt")
    a.save_checkpoint(path, global_step=1)
    off = p2r.Model(cfg, 99, offload=[1, 0, 1], ring_slots=2)
    off.load_checkpoint(path)
    pa, po = a.params(), off.params()
    for n in a.names:
        assert np.array_equal(pa[n], po[n]), n
    off.set_offload_lr(1e-3 * 2)
    tok, tgt, mask = lm_batch(8, 128, 12)
    la = a.train_step(tok, tgt, mask, 8, float(mask.sum()))
    a.adamw_step(1e-3 * 2)
    lo = off.train_step(tok, tgt, mask, 8, float(mask.sum()))
    off.adamw_step(1e-3 * 2)
    assert la == lo
    assert_same_state(a, off)


def test_redistribute_experts(cuda, tmp_path):
    """SPEC redistribute_experts (model.cpp:334-356): in-process re-sharding is bookkeeping
    with identical outputs; across GPU counts the shard checkpoints carry each expert's
    weights and moments to its new owner, and 1 -> 2 -> 1 restores the model bitwise."""
    import paper_2110_03888_b200 as p2r
    m = p2r.Model(p2r.Config(**C1), 1234)
    m.attach_adamw()
    step(m, 0, seed=21)
    tok, _, _ = lm_batch(8, 128, seed=22)
    before = m.forward(tok, 8)
    assert m.shard_layout() == [[0, 1, 2, 3]]
    m.redistribute_experts(2)
    assert m.shard_layout() == [[0, 1], [2, 3]] and m.expert_shard(3) == 1
    assert np.array_equal(m.forward(tok, 8), before)
    with pytest.raises(p2r.P2RInvalidArgument, match="divisible by new shard count"):
        m.redistribute_experts(3)
    with pytest.raises(p2r.P2ROutOfRange, match="expert index"):
        m.expert_shard(4)
    m.redistribute_experts(1)
    full = str(tmp_path / "full.p2rckpt")
    m.save_checkpoint(full, global_step=1)
    shards = [str(tmp_path / f"s{r}.p2rckpt") for r in range(2)]
    p2r.redistribute_checkpoints([full], shards)
    pm, mm = m.params(), m.moments()
    for r, path in enumerate(shards):
        sh, st = p2r.load_checkpoint(path)  # an expert-parallel shard model (ep = (2, r))
        assert st["global_step"] == 1 and sh.step_count() == m.step_count()
        ps, ms = sh.params(), sh.moments()
        experts = sorted({int(n.split(".")[4]) for n in ps if ".moe.expert." in n})
        assert experts == [2 * r, 2 * r + 1]
        for n in ps:
            assert np.array_equal(ps[n], pm[n]), n
            assert np.array_equal(ms[n][0], mm[n][0]) and np.array_equal(ms[n][1], mm[n][1]), n
        sh.close()
    back = str(tmp_path / "back.p2rckpt")
    p2r.redistribute_checkpoints(shards, [back])
    b, _ = p2r.load_checkpoint(back)
    assert_same_state(m, b)
    assert np.array_equal(b.forward(tok, 8), before)


def test_load_without_optimizer_state_resets_moments(cuda, tmp_path):
    """a snapshot taken before the optimizer existed restores a fresh
    optimizer (zero moments, step 0), and saves go through a temporary + rename."""
    import os

    import paper_2110_03888_b200 as p2r
    a = p2r.Model(p2r.Config(**REAL), 1234)
    path = str(tmp_path / "no_opt.p2rckpt")
    a.save_checkpoint(path)
    assert not os.path.exists(path + ".tmp")
    a.attach_adamw()
    step(a, 0, seed=5)
    a.load_checkpoint(path)
    assert a.step_count() == 0
    for n, (m, v) in a.moments().items():
        assert not m.any() and not v.any(), n
    b = p2r.Model(p2r.Config(**REAL), 1234)
    b.attach_adamw()
    assert_same_state(a, b)
    assert step(a, 0, seed=6) == step(b, 0, seed=6)
    assert_same_state(a, b)
