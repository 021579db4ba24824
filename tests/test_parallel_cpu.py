"""CPU, world_size 2 over gloo: the multi-GPU host logic of the step.

* DP: each rank runs its own micro-batch with the GLOBAL mask count as the CE
  denominator and the replicated gradients are summed — equal to the
  single-process large-batch gradient (tensor.hpp:135-140).
* EP: the expert-segment exchange layout the engine uses (csrc/engine/comm.cpp,
  Model::ep_exchange: local [E][seg] <-> owner [El][W][seg], rank r owning
  experts [r*El, (r+1)*El) as Model::expert_shard, model.cpp:334-340), with
  per-rank routing/capacity on the rank's own tokens, reproduces
  the single-process MoE sublayer on every rank's tokens.
The oracle restatement is the checker; gloo carries the exchange."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import p2r_oracle as O

TINY = dict(d_model=32, d_ff=64, n_layers_graph=3, n_layers_params=1, n_heads=2, vocab_size=260, seq_len=16)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def lm_batch(batch, seq, seed):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok, tgt, mask


def params_for(cfg):
    golden = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "tiny_dense.npz")))
    return {k[3:]: v for k, v in golden.items() if k.startswith("p0.")}


def _dp_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = O.Config(**TINY)
    tok, tgt, mask = lm_batch(4, 16, 5)
    denom = float(mask.sum())  # global count over all ranks' micro-batches
    sl = slice(rank * 2, rank * 2 + 2)
    m = O.Model(cfg, params_for(cfg))
    loss, G = m.loss_and_grads(tok[sl].ravel(), tgt[sl].ravel(), mask[sl].ravel(), 2, denom)
    lt = torch.tensor([loss], dtype=torch.float64)
    dist.all_reduce(lt)
    for k in sorted(G):
        t = torch.from_numpy(G[k].copy())
        dist.all_reduce(t)
        G[k] = t.numpy()
    if rank == 0:
        full = O.Model(cfg, params_for(cfg))
        lf, Gf = full.loss_and_grads(tok.ravel(), tgt.ravel(), mask.ravel(), 4, denom)
        worst = max(float(np.linalg.norm(G[k] - Gf[k]) / (np.linalg.norm(Gf[k]) + 1e-30)) for k in Gf)
        out.put((float(lt.item()), lf, worst))
    dist.destroy_process_group()


def test_dp_allreduce_equals_large_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ctx_procs = [ctx.Process(target=_dp_worker, args=(r, 2, free_port_cached(), q)) for r in range(2)]
    for p in ctx_procs:
        p.start()
    loss_sum, loss_full, worst = q.get(timeout=240)
    for p in ctx_procs:
        p.join(timeout=60)
    assert abs(loss_sum - loss_full) <= 1e-5 * abs(loss_full)
    assert worst < 1e-5


_PORT = None


def free_port_cached():
    global _PORT
    if _PORT is None:
        _PORT = free_port()
    return _PORT


# ---------------------------------------------------------------- EP protocol
E, K, D, FF = 4, 1, 8, 16


def _expert(x, w1, b1, w2, b2):
    return (O.gelu_fwd((x @ w1 + b1).astype(np.float32)) @ w2 + b2).astype(np.float32)


def _ep_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(123)  # same weights on every rank
    W1 = rng.standard_normal((E, D, FF)).astype(np.float32) * 0.3
    B1 = rng.standard_normal((E, FF)).astype(np.float32) * 0.1
    W2 = rng.standard_normal((E, FF, D)).astype(np.float32) * 0.3
    B2 = rng.standard_normal((E, D)).astype(np.float32) * 0.1
    T = 40
    rr = np.random.default_rng(1000 + rank)  # rank-local tokens and gate logits
    b = rr.standard_normal((T, D)).astype(np.float32)
    logits = rr.standard_normal((T, E)).astype(np.float32)
    logits[:, 0] += 0.8  # skewed -> capacity drops
    r = O.moe_dispatch(logits, E, K, 1.0)  # per-rank routing on the rank's own tokens
    cap = r.capacity
    seg = min(cap, T)
    El = E // world
    # dispatch into the local expert-major layout [E][seg] (zero padding)
    local = np.zeros((E, seg, D), np.float32)
    for e in range(E):
        for i, t in enumerate(r.expert_rows[e]):
            local[e, i] = b[t]
    # ep_exchange(to_experts): peer q receives my blocks e in [q*El, (q+1)*El) into
    # its owner layout [El][W][seg] at position (e_local*W + my_rank)
    send = np.concatenate([local[q * El:(q + 1) * El].reshape(-1) for q in range(world)])
    recv = torch.empty(send.size, dtype=torch.float32)
    dist.all_to_all_single(recv, torch.from_numpy(send))
    chunks = recv.numpy().reshape(world, El, seg, D)  # [source q][e_local]
    owner = np.zeros((El, world, seg, D), np.float32)
    for q in range(world):
        for el in range(El):
            owner[el, q] = chunks[q, el]
    # owner-side expert FFN with the global expert index rank*El + el
    y_owner = np.zeros_like(owner)
    for el in range(El):
        e = rank * El + el
        y_owner[el] = _expert(owner[el].reshape(-1, D), W1[e], B1[e], W2[e], B2[e]).reshape(world, seg, D)
    # ep_exchange(combine): send owner block (el, q) back to q
    send2 = np.concatenate([y_owner[:, q].reshape(-1) for q in range(world)])
    recv2 = torch.empty(send2.size, dtype=torch.float32)
    dist.all_to_all_single(recv2, torch.from_numpy(send2))
    back = recv2.numpy().reshape(world, El, seg, D)  # [owner q][e_local] -> global expert q*El + el
    ye = back.reshape(E, seg, D)
    # combine (weights are exactly 1 for top-1) vs the single-process expert math
    out_ep = np.zeros((T, D), np.float32)
    ref = np.zeros((T, D), np.float32)
    for e in range(E):
        rows = r.expert_rows[e]
        if len(rows):
            out_ep[rows] += ye[e, :len(rows)]
            ref[rows] += _expert(b[rows], W1[e], B1[e], W2[e], B2[e])
    out.put((rank, float(np.abs(out_ep - ref).max()), r.dropped))
    dist.destroy_process_group()


def test_ep_exchange_layout_reproduces_single_process_moe():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, dropped in res:
        assert err < 1e-5, (rank, err)
    assert sum(d for _, _, d in res) > 0  # the case exercises capacity drops
