"""ORACLE / TEST INFRASTRUCTURE ONLY — generates tests/golden/*.npz from the
compiled reference (oracle/_ref/libp2r_ref.so, built from /root/reference by
oracle/build_ref.sh). Run here (where /root/reference exists):

    bash oracle/build_ref.sh && python oracle/make_goldens.py

The fixtures pin both the numpy restatement (oracle/p2r_oracle.py) and the
CUDA path; they are small enough to commit.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import ref  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden")

TINY_DENSE = dict(d_model=32, d_ff=64, n_layers_graph=3, n_layers_params=1, n_heads=2,
                  vocab_size=260, seq_len=16, n_experts=0, n_prototypes=1)
TINY_MOE = dict(d_model=32, d_ff=64, n_layers_graph=3, n_layers_params=1, n_heads=2,
                vocab_size=260, seq_len=16, n_experts=4, n_prototypes=2, capacity_factor=1.0)
C1 = dict(d_model=256, d_ff=1024, n_layers_graph=4, n_layers_params=1, n_heads=4,
          vocab_size=260, seq_len=128, n_experts=4, n_prototypes=1)


def lm_batch(batch, seq, seed=7):
    """Synthetic LM batch with make_lm_batch semantics (data.cpp:174-195):
    targets = next token, mask = 1 except the last position."""
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


def step_fixture(name, cfgd, batch, seq, full=True):
    cfg = ref.Config(**cfgd)
    m = ref.RefModel(cfg, 1234)
    p0 = m.params()
    tok, tgt, mask = lm_batch(batch, seq)
    denom = float(mask.sum())
    m.attach_adamw()
    logits0 = m.forward(tok, batch)
    loss = m.train_step(tok, tgt, mask, batch, denom)
    g = m.grads()
    lr = 2e-4
    m.adamw_step(lr)
    p1 = m.params()
    mom = m.moments()
    d = {"tokens": tok, "targets": tgt, "mask": mask, "batch": np.int32(batch),
         "loss": np.float32(loss), "lr": np.float32(lr), "denom": np.float64(denom)}
    for k in sorted(cfgd):
        d["cfg." + k] = np.asarray(cfgd[k])
    if full:
        d["logits0"] = logits0
        for n in m.names:
            d["p0." + n] = p0[n]
            d["g." + n] = g[n]
            d["p1." + n] = p1[n]
            d["m." + n] = mom[n][0]
            d["v." + n] = mom[n][1]
        # delink of the post-step model: bitwise logits equality
        real = m.delinked()
        d["delinked_logits"] = real.forward(tok, batch)
        d["pseudo_logits"] = m.forward(tok, batch)
    else:
        rng = np.random.default_rng(0)
        for n in m.names:
            flat = g[n].ravel()
            idx = rng.choice(flat.size, size=min(64, flat.size), replace=False).astype(np.int64)
            d["gnorm." + n] = np.float64(np.linalg.norm(flat.astype(np.float64)))
            d["gidx." + n] = idx
            d["gval." + n] = flat[idx]
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
    print(name, "loss", loss)


def routing_fixtures():
    d = {}
    # SPEC / survey KAT: capacity 1, selected 0 1 0 0, survived 1 1 0 0, dropped 2
    kat = np.array([[1, 1, 0, 0], [0, 2, 2, 0], [5, 0, 0, 0], [3, 3, 3, 3]], np.float32)
    r = ref.moe_dispatch(kat, 4, 1, 1.0)
    d.update({"kat.logits": kat, "kat.selected": r.selected, "kat.survived": r.survived,
              "kat.capacity": np.int32(r.capacity), "kat.dropped": np.int32(r.dropped),
              "kat.offsets": r.offsets, "kat.rows": r.rows, "kat.slots": r.slots,
              "kat.raw_load": r.raw_load})
    # randomized cases incl. ties, NaN, drops, k=2, E=64
    rng = np.random.default_rng(11)
    cases = [(1024, 4, 1, 1.25), (1024, 4, 1, 1.0), (257, 8, 2, 1.0), (2048, 64, 1, 1.25),
             (500, 16, 4, 0.5)]
    for i, (T, E, k, cf) in enumerate(cases):
        lg = rng.standard_normal((T, E)).astype(np.float32)
        if i == 1:
            lg = np.round(lg)  # many exact ties
        if i == 2:
            lg[rng.integers(0, T, 20), rng.integers(0, E, 20)] = np.nan
        if i == 4:
            lg[:, 0] += 3.0  # skew -> heavy drops
        r = ref.moe_dispatch(lg, E, k, cf)
        pre = f"c{i}."
        d.update({pre + "logits": lg, pre + "E": np.int32(E), pre + "k": np.int32(k),
                  pre + "cf": np.float32(cf), pre + "selected": r.selected,
                  pre + "survived": r.survived, pre + "raw_load": r.raw_load,
                  pre + "offsets": r.offsets, pre + "rows": r.rows, pre + "slots": r.slots,
                  pre + "capacity": np.int32(r.capacity), pre + "dropped": np.int32(r.dropped)})
    np.savez_compressed(os.path.join(OUT, "routing.npz"), **d)
    print("routing cases", len(cases) + 1)


def primitive_fixtures():
    rng = np.random.default_rng(3)
    d = {}
    x = rng.standard_normal((6, 40)).astype(np.float32)
    x[0] = 5.0  # constant row -> 0
    gain = rng.standard_normal(40).astype(np.float32)
    bias = rng.standard_normal(40).astype(np.float32)
    gy = rng.standard_normal((6, 40)).astype(np.float32)
    y, gx, gg, gb = ref.layernorm(x, gain, bias, gy)
    d.update({"ln.x": x, "ln.gain": gain, "ln.bias": bias, "ln.gy": gy, "ln.y": y, "ln.gx": gx,
              "ln.ggain": gg, "ln.gbias": gb})
    q, k, v, go = (rng.standard_normal((2, 2, 24, 16)).astype(np.float32) for _ in range(4))
    for causal in (0, 1):
        o, gq, gk, gv = ref.attention(q, k, v, go, bool(causal))
        d.update({f"att{causal}.o": o, f"att{causal}.gq": gq, f"att{causal}.gk": gk,
                  f"att{causal}.gv": gv})
    d.update({"att.q": q, "att.k": k, "att.v": v, "att.go": go})
    lg = (3 * rng.standard_normal((9, 260))).astype(np.float32)
    tg = rng.integers(0, 260, 9).astype(np.int32)
    mk = (rng.random(9) > 0.3).astype(np.uint8)
    loss, g = ref.cross_entropy(lg, tg, mk, 17.0)
    d.update({"ce.logits": lg, "ce.targets": tg, "ce.mask": mk, "ce.denom": np.float64(17.0),
              "ce.loss": np.float32(loss), "ce.glogits": g})
    xs = np.linspace(-6, 6, 301).astype(np.float32)
    gys = rng.standard_normal(301).astype(np.float32)
    y, gx = ref.gelu(xs, gys)
    d.update({"gelu.x": xs, "gelu.gy": gys, "gelu.y": y, "gelu.gx": gx})
    # LR schedule (optim.cpp:8-24)
    steps = np.arange(0, 120, dtype=np.int64)
    d["lr.steps"] = steps
    d["lr.values"] = np.array([ref.lr_at(2e-4, 0.1, 100, int(s)) for s in steps], np.float32)
    # count_params (model.cpp:73-89) for the SPEC Table-1 configs and C1..C4
    cfgs = {
        "pseudo": dict(d_model=1024, d_ff=16384, n_layers_graph=36, n_layers_params=1, n_heads=16, vocab_size=50000, seq_len=512),
        "real": dict(d_model=1024, d_ff=16384, n_layers_graph=36, n_layers_params=36, n_heads=16, vocab_size=50000, seq_len=512),
        "base": dict(d_model=1024, d_ff=4096, n_layers_graph=24, n_layers_params=24, n_heads=16, vocab_size=50000, seq_len=512),
        "c1": C1,
    }
    for k_, c in cfgs.items():
        d["count." + k_] = np.array(ref.count_params(ref.Config(**c)), np.int64)
    np.savez_compressed(os.path.join(OUT, "primitives.npz"), **d)
    print("primitives ok")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    step_fixture("tiny_dense", TINY_DENSE, 2, 16)
    step_fixture("tiny_moe", TINY_MOE, 2, 16)
    step_fixture("c1", C1, 8, 128, full=False)
    routing_fixtures()
    primitive_fixtures()
