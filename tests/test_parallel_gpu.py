"""Expert / data parallelism on one B200 (the only GPU this run has).

* World size 1: the expert-parallel exchange path (peer-store send -> owner pack
  -> exact-count grouped GEMMs -> peer-store return, csrc/ep.cu), forced with
  P2R_FORCE_EP=1, gives the same bits as the local path; a world-of-one NCCL
  all-reduce leaves the gradients unchanged.
* World size 2 and 4: W shards of this process on the device, one host thread
  each (LoopbackGroup), run the SAME exchange kernels and stream flags as the
  multi-GPU path with the shards' arenas as the peer memory. Every expert row is
  computed row-independently, so each rank's loss and the gradient flowing into
  its replicated layers are bitwise those of a full model run on that rank's
  tokens; the rank-order all-reduce then equals the fp32 sum of those models'
  gradients bit for bit, and each owner's expert gradients equal the sum over all
  sources (summation order differs: <= 1e-5).
Multi-rank host logic over gloo: tests/test_parallel_cpu.py."""
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


def _run_ranks(fns):
    """Run one callable per shard on its own thread (the exchange is collective)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(fns)) as ex:
        futs = [ex.submit(f) for f in fns]
        return [f.result(timeout=600) for f in futs]


MOE_W = dict(d_model=256, d_ff=512, n_layers_graph=3, n_layers_params=3, n_heads=4, vocab_size=260,
             seq_len=128, n_experts=8, n_prototypes=1)


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("cfgd", [MOE_W, dict(MOE_W, n_layers_params=1),
                                  dict(MOE_W, n_prototypes=2, capacity_factor=1.0),
                                  dict(MOE_W, n_experts=0)],
                         ids=["real_top1", "pseudo_top1", "real_k2_drops", "dense_dp"])
def test_loopback_ranks_match_full_models(cuda, W, cfgd):
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**cfgd)
    B, S = 2, 128
    batches = [lm_batch(B, S, seed=40 + r) for r in range(W)]
    denom = float(sum(b[2].sum() for b in batches))  # global mask count
    group = p2r.LoopbackGroup(W)
    shards = [p2r.Model(cfg, 1234, ep=(W, r)) for r in range(W)]
    for m in shards:
        m.comm_init_loopback(group)
    full = [p2r.Model(cfg, 1234) for _ in range(W)]
    for step in range(2):
        def rank_step(r):
            tok, tgt, mask = batches[r]
            loss = shards[r].train_step(tok, tgt, mask, B, denom)
            shards[r].allreduce_grads()
            return loss

        losses = _run_ranks([lambda r=r: rank_step(r) for r in range(W)])
        ref = [full[r].train_step(*batches[r], B, denom) for r in range(W)]
        assert losses == ref, (losses, ref)
        gfull = [f.grads() for f in full]
        for r, m in enumerate(shards):
            gs = m.grads()
            for n, v in gs.items():
                if ".moe.expert." in n:
                    e = int(n.split(".")[4])
                    assert e // (cfgd["n_experts"] // W) == r, n  # the owner holds it
                    want = sum(g[n].astype(np.float64) for g in gfull)
                    den = np.linalg.norm(want)
                    err = np.linalg.norm(v - want) / den if den > 0 else np.abs(v).max()
                    assert err <= 1e-5, (n, err)
                else:  # replicated: rank-order fp32 sum of the full models' grads, bitwise
                    want = gfull[0][n].copy()
                    for g in gfull[1:]:
                        want = (want + g[n]).astype(np.float32)
                    assert np.array_equal(v, want), (r, n)
    for m in shards:
        m.close()


def test_loopback_ep_offload_accumulation_matches_resident(cuda):
    """C5's engine shape at W=2: expert-parallel shards with SLOW layer granules
    (offload + activation checkpointing + 2-micro-step accumulation, the SLOW
    replicated grads all-reduced inside the backward) train bit-identically to
    the resident expert-parallel shards."""
    import paper_2110_03888_b200 as p2r
    W, B, S = 2, 2, 128
    cfg = p2r.Config(**dict(MOE_W, n_layers_graph=4, n_layers_params=4))
    runs = []
    for offload in (None, [1, 0, 1, 1]):
        group = p2r.LoopbackGroup(W)
        shards = [p2r.Model(cfg, 1234, ep=(W, r), offload=offload, ring_slots=2) for r in range(W)]
        for m in shards:
            m.comm_init_loopback(group)
            m.attach_adamw()
            if offload:
                m.set_grad_accumulation(2)

        def rank_run(r):
            m = shards[r]
            out = []
            for step in range(2):
                lr = 1e-3 * (step + 1)
                if offload:
                    m.set_offload_lr(lr)
                for micro in range(2):
                    tok, tgt, mask = lm_batch(B, S, seed=100 + 10 * step + 2 * micro + r)
                    out.append(m.train_step(tok, tgt, mask, B, 4.0 * W * (B * (S - 1)), zero=(micro == 0)))
                m.allreduce_grads()
                m.adamw_step(lr)
            return out

        losses = _run_ranks([lambda r=r: rank_run(r) for r in range(W)])
        runs.append((losses, [m.params() for m in shards]))
    assert runs[0][0] == runs[1][0]
    for r in range(W):
        for n, v in runs[0][1][r].items():
            assert np.array_equal(v, runs[1][1][r][n]), (r, n)


@pytest.mark.parametrize("cfgd", [MOE_W, dict(MOE_W, n_experts=0)], ids=["ep_moe", "dense_dp"])
def test_loopback_pipelined_host_steps_bit_identical(cuda, cfgd):
    """Model.train_step(wait=False) on expert-parallel / data-parallel loopback shards (the
    exchange and the all-reduce are collective, each shard on its own host thread): the
    next step and the all-reduce are enqueued before the previous loss is read; losses and
    gradients are bit-identical to the synchronous loop."""
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(**cfgd)
    W, B, S, steps = 2, 2, 128, 3
    batches = [[lm_batch(B, S, seed=60 + 10 * r + i) for i in range(steps)] for r in range(W)]
    denom = float(sum(b[2].sum() for b in batches[0]))
    out = {}
    for piped in (False, True):
        group = p2r.LoopbackGroup(W)
        shards = [p2r.Model(cfg, 1234, ep=(W, r)) for r in range(W)]
        for m in shards:
            m.comm_init_loopback(group)

        def run(r):
            losses, prev = [], None
            for i in range(steps):
                tok, tgt, mask = batches[r][i]
                if piped:
                    cur = shards[r].train_step(tok, tgt, mask, B, denom, wait=False)
                    shards[r].allreduce_grads()
                    if prev is not None:
                        losses.append(prev.value())
                    prev = cur
                else:
                    losses.append(shards[r].train_step(tok, tgt, mask, B, denom))
                    shards[r].allreduce_grads()
            if piped:
                losses.append(prev.value())
            return losses

        losses = _run_ranks([lambda r=r: run(r) for r in range(W)])
        out[piped] = (losses, [m.grads() for m in shards])
        for m in shards:
            m.close()
    assert out[True][0] == out[False][0]
    for r in range(W):
        for n, v in out[False][1][r].items():
            assert np.array_equal(v, out[True][1][r][n]), (r, n)
