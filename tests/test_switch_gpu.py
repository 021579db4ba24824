"""Live switch-detector evaluation on the B200: snapshot ->
delink -> Real trial -> revert -> Pseudo continuation. Revert correctness: the
Pseudo model after the evaluation equals, bit for bit, a twin that skipped the
trial and trained the same number of steps from the snapshot."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C1 = dict(d_model=256, d_ff=1024, n_layers_graph=4, n_layers_params=1, n_heads=4, vocab_size=260,
          seq_len=128, n_experts=4, n_prototypes=1)


def lm_batch(seed):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (8, 128)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


def test_switch_evaluation_reverts_exactly(cuda, tmp_path):
    import paper_2110_03888_b200 as p2r
    from paper_2110_03888_b200.switch import SwitchDetector, SwitchPolicy

    class Clock:  # one tick per training step: the continuation runs exactly the trial length
        def __init__(self):
            self.t = 0.0

        def __call__(self):
            return self.t

    clock = Clock()
    counters = {}

    def step_fn(m):
        k = counters.get(id(m), 0)
        counters[id(m)] = k + 1
        tok, tgt, mask = lm_batch(1000 + k)
        m.train_step(tok, tgt, mask, 8, float(mask.sum()))
        m.adamw_step(1e-3)
        clock.t += 1.0

    eval_batch = lm_batch(7)

    def eval_fn(m):
        tok, tgt, mask = eval_batch
        logits = m.forward(tok, 8).reshape(-1, 260).astype(np.float64)
        logits -= logits.max(1, keepdims=True)
        lp = logits - np.log(np.exp(logits).sum(1, keepdims=True))
        nll = -lp[np.arange(len(tgt)), tgt]
        return float((nll * mask).sum() / mask.sum())

    m = p2r.Model(p2r.Config(**C1), 1234)
    m.attach_adamw()
    for k in range(4):
        tok, tgt, mask = lm_batch(k)
        m.train_step(tok, tgt, mask, 8, float(mask.sum()))
        m.adamw_step(1e-3)
    snap = str(tmp_path / "twin.p2rckpt")
    m.save_checkpoint(snap, global_step=4)
    twin, _ = p2r.load_checkpoint(snap)

    det = SwitchDetector(SwitchPolicy(eval_interval_steps=4, trial_budget_steps=4, slope_window=4), clock=clock)
    assert det.due(4) and not det.due(3)
    res = det.evaluate(m, step_fn, eval_fn, str(tmp_path / "snap.p2rckpt"), step=4)
    assert res["pseudo_steps"] == 4 and res["trial_s"] == 4.0
    assert isinstance(res["fire"], bool) and np.isfinite(res["pseudo_slope"]) and np.isfinite(res["real_slope"])
    # the twin trains the same 4 continuation batches: bit-identical to the evaluated model
    counters[id(twin)] = counters[id(m)] - 4
    for _ in range(4):
        step_fn(twin)
    pa, pb = m.params(), twin.params()
    for n in m.names:
        assert np.array_equal(pa[n], pb[n]), n
    assert m.step_count() == twin.step_count()
