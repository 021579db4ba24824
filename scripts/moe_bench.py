"""MoE training-step throughput on one B200 at the C4 per-rank shape:
d = 2048, 16 heads (hd 128), d_ff = 4096, top-1 over E local experts (E = 8 = C4's 64
experts / 8 ranks, so each GPU's expert GEMMs see the same rows as under EP-8; the
expert all-to-all itself needs 8 GPUs and is not in this number), 8 x 1024 tokens per
step, `--layers` delinked (Real) layers, fwd + bwd + AdamW. Wall time of K steps between
device-wide synchronisations, after W warm-up steps; model FLOPs per §8(d) with k_eff = admitted rows / T.

  python scripts/moe_bench.py [--layers 4 --experts 8 --steps 10 --warmup 3 --out f.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--dff", type=int, default=4096)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(d_model=a.d, d_ff=a.dff, n_layers_graph=a.layers, n_layers_params=a.layers, n_heads=a.heads,
                     vocab_size=260, seq_len=a.seq, n_experts=a.experts, n_prototypes=1)
    m = p2r.Model(cfg, 1234)
    m.attach_adamw()
    B, S = a.batch, a.seq
    rng = np.random.default_rng(7)
    tok = rng.integers(0, 256, (B, S)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    dt, dg, dm = (torch.from_numpy(x.ravel()).cuda() for x in (tok, tgt, mask))
    denom = float(mask.sum())

    def step(i):
        m.train_step_device(dt.data_ptr(), dg.data_ptr(), dm.data_ptr(), B, S, denom)
        m.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, i + 10))

    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize()
    n0 = p2r.launch_count()
    # the model runs on its own stream: time with device-wide synchronisation on both sides
    t0 = time.perf_counter()
    for i in range(a.steps):
        step(a.warmup + i)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / a.steps
    launches = (p2r.launch_count() - n0) / a.steps
    T, d, dff, E, L = B * S, a.d, a.dff, a.experts, a.layers
    cap = p2r.lib().p2r_moe_capacity(__import__("ctypes").c_float(1.25), T, E, 1)
    k_eff = min(1.0, cap * E / T)  # upper bound on admitted rows / T (drops are rare at cf 1.25)
    f_tok = 3 * (L * (8 * d * d + 4 * k_eff * d * dff + 2 * d * E + 2 * S * d) + 2 * d * 260)
    tps = T / (ms / 1e3)
    out = {"workload": f"Real MoE L={L} d={d} heads={a.heads} d_ff={dff} E={E} top-1 cf 1.25, {B}x{S} tokens/step, "
                       "fwd+bwd+AdamW, 1 GPU (C4 per-rank expert rows, no all-to-all)",
           "ms_per_step": round(ms, 3), "tokens_per_s": round(tps, 1),
           "model_tflops": round(f_tok * tps / 1e12, 1), "model_flops_per_token": f_tok,
           "kernel_launches_per_step": launches, "steps": a.steps, "warmup": a.warmup}
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
