"""NCCL paths on one B200 (the only GPU this run has). A world-size-1
communicator still runs the real code: the expert-parallel exchange path
(grouped ncclSend/ncclRecv of fixed-capacity expert segments + full-capacity
grouped GEMMs on the owner layout), forced with P2R_FORCE_EP=1, must give the
same bits as the local path; the DP all-reduce must leave a single rank's
gradients unchanged. Multi-rank layout / DP math: tests/test_parallel_cpu.py."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

C1 = dict(d_model=256, d_ff=1024, n_layers_graph=4, n_layers_params=1, n_heads=4, vocab_size=260,
          seq_len=128, n_experts=4, n_prototypes=1)


def lm_batch(batch, seq, seed=7):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


@pytest.mark.parametrize("cfgd", [C1, dict(C1, n_layers_params=4, n_experts=8, n_prototypes=2, capacity_factor=1.0)],
                         ids=["pseudo_top1", "real_k2"])
def test_ep_exchange_path_bit_identical(cuda, cfgd):
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**cfgd)
    ref = p2r.Model(cfg, 1234)
    os.environ["P2R_FORCE_EP"] = "1"
    try:
        ep = p2r.Model(cfg, 1234, ep=(1, 0))
    finally:
        del os.environ["P2R_FORCE_EP"]
    with pytest.raises(p2r.P2RLogicError, match="comm_init"):
        tok, tgt, mask = lm_batch(8, 128)
        ep.train_step(tok, tgt, mask, 8, float(mask.sum()))
    ep.comm_init(p2r.comm_unique_id())
    tok, tgt, mask = lm_batch(8, 128)
    a = ref.train_step(tok, tgt, mask, 8, float(mask.sum()))
    b = ep.train_step(tok, tgt, mask, 8, float(mask.sum()))
    assert a == b
    ga, gb = ref.grads(), ep.grads()
    for n in ga:
        assert np.array_equal(ga[n], gb[n]), n
    ep.allreduce_grads()  # world of one: sum over one rank
    gc = ep.grads()
    for n in ga:
        assert np.array_equal(ga[n], gc[n]), n


def test_ep_shard_holds_its_experts(cuda):
    """Rank r of W holds experts [r*E/W, (r+1)*E/W) with the reference's init bits."""
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**dict(C1, n_experts=8))
    full = p2r.Model(cfg, 1234)
    shard = p2r.Model(cfg, 1234, ep=(4, 2))
    names = [n for n in shard.names if ".moe.expert." in n]
    assert sorted({int(n.split(".")[4]) for n in names}) == [4, 5]
    pf, ps = full.params(), shard.params()
    for n in ps:
        assert np.array_equal(pf[n], ps[n]), n


def test_dp_graph_step_then_allreduce_bit_identical(cuda):
    """A dense data-parallel model (communicator initialised) replays its step as a CUDA
    graph; the all-reduce follows on the same stream; grads match the eager path."""
    import torch
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(d_model=256, d_ff=1024, n_layers_graph=3, n_layers_params=1, n_heads=4, vocab_size=260,
                     seq_len=128)
    tok, tgt, mask = (torch.from_numpy(a).cuda() for a in lm_batch(8, 128))
    grads = []
    for graph in (False, True):
        m = p2r.Model(cfg, 1234)
        m.comm_init(p2r.comm_unique_id())
        for _ in range(3):
            m.train_step_device(tok.data_ptr(), tgt.data_ptr(), mask.data_ptr(), 8, 128, 1016.0, graph=graph)
            m.allreduce_grads()
        torch.cuda.synchronize()
        grads.append(m.grads())
        m.close()
    for n in grads[0]:
        assert np.array_equal(grads[0][n], grads[1][n]), n
