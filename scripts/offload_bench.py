"""Granular-offload measurement on one B200 (§4.2).

Real dense stack (default d=2048, d_ff=8192, 16 layers, 16 x 1024 tokens per
step) trained three ways with identical kernels:
  resident : every layer granule in HBM                      -> compute-only time
  offload  : the planner's SLOW layers in pinned host DRAM, streamed through
             HBM staging slots one granule ahead on H2D / D2H side streams
  no-copy  : the offload schedule with the PCIe copies skipped (same waits)
and reports bytes per phase, measured PCIe GB/s per direction, and the hidden
fraction h = 1 - (T_offload - T_nocopy) / max(T_h2d, T_d2h).

  python scripts/offload_bench.py [--layers 16 --d 2048 --dff 8192 --batch 16 --plan interleave]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lm_batch(batch, seq, seed):
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


def overlap_prediction(p2r, rec, L):
    """predict_step_time_overlap from a bench record: measured per-direction PCIe rates,
    per-layer compute from the resident step (forward : backward = 1 : 2)."""
    P = rec["granule_bytes_18B_per_param"] // 18
    n_slow = rec["slow_layers"]
    vec = max(0, (rec["bytes_per_step"]["Fn_load"] / max(1, n_slow) - 2 * P) / 4)
    t = rec["step_s"]["resident"] / L
    return p2r.predict_step_time_overlap([P] * L, rec["placement"], rec["h2d_GBps"] * 1e9, rec["d2h_GBps"] * 1e9,
                                         t / 3, 2 * t / 3, vector_params=[int(vec)] * L,
                                         fn_master=rec.get("fn_form", "shadow") == "master")


def run(model, p2r, args, steps, offloaded):
    import torch
    B, S = args.batch, args.seq
    tok, tgt, mask = lm_batch(B, S, 7)
    dt = torch.from_numpy(tok).cuda()
    dg = torch.from_numpy(tgt).cuda()
    dm = torch.from_numpy(mask).cuda()
    denom = float(mask.sum())

    def one(i):
        lr = p2r.lr_at(2e-4, 0.01, 1000, i + 10)
        if offloaded:
            model.set_offload_lr(lr)
        model.train_step_device(dt.data_ptr(), dg.data_ptr(), dm.data_ptr(), B, S, denom)
        model.adamw_step(lr)

    for i in range(2):
        one(i)
    torch.cuda.synchronize()
    if offloaded:
        model.offload_stats()  # drains the copy streams
        model.offload_stats_reset()
    t0 = time.perf_counter()
    for i in range(steps):
        one(2 + i)
    stats = model.offload_stats() if offloaded else None  # waits for the last write-backs
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps, stats


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--d", type=int, default=2048)
    ap.add_argument("--dff", type=int, default=8192)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--ring", type=int, default=3)
    ap.add_argument("--plan", default="interleave", choices=["interleave", "prefix"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "offload_r01.json"))
    args = ap.parse_args()
    import torch
    import paper_2110_03888_b200 as p2r
    cfg = p2r.Config(d_model=args.d, d_ff=args.dff, n_layers_graph=args.layers, n_layers_params=args.layers,
                     n_heads=args.heads, vocab_size=260, seq_len=args.seq)
    L = args.layers
    if args.plan == "interleave":
        plan = [1 if i % 2 == 0 else 0 for i in range(L)]
    else:
        # SPEC planner: uniform layers, half-model budget -> the first L/2 layers (§4.2)
        gb = 18 * p2r.count_params(cfg)[1]
        plan = p2r.plan_offload([gb] * L, gb * (L - L // 2), 50e9, 1.0)

    res = p2r.Model(cfg, 1234)
    res.attach_adamw()
    t_res, _ = run(res, p2r, args, args.steps, False)
    res.close()
    del res
    torch.cuda.empty_cache()

    off = p2r.Model(cfg, 1234, offload=plan, ring_slots=args.ring)
    off.attach_adamw()
    t_off, st = run(off, p2r, args, args.steps, True)
    off.set_offload_skip_copies(True)
    t_nocopy, _ = run(off, p2r, args, args.steps, True)
    off.set_offload_skip_copies(False)

    per = {k: v / args.steps for k, v in st.items()}
    h2d_b = per["Fn_load"] + per["Bn_load"] + per["opt_load"]
    d2h_b = per["writeback"] + per["grad_offload"]
    t_copy = max(per["h2d_ms"], per["d2h_ms"]) / 1e3
    hidden = 1.0 - max(0.0, t_off - t_nocopy) / t_copy if t_copy > 0 else 1.0
    T = args.batch * args.seq
    gran = off.layer_granule_bytes()
    out = {
        "workload": f"Real dense stack L={L} d={args.d} d_ff={args.dff} heads={args.heads}, {args.batch}x{args.seq} tokens/step, fwd+bwd+AdamW",
        "placement": plan, "slow_layers": int(sum(plan)), "ring_slots": args.ring,
        "fn_form": "shadow" if os.environ.get("P2R_OFFLOAD_FN_SHADOW") == "1" else "master",
        "granule_bytes_18B_per_param": gran,
        "step_s": {"resident": round(t_res, 4), "offload": round(t_off, 4), "offload_no_copy": round(t_nocopy, 4)},
        "bytes_per_step": {k: per[k] for k in ("Fn_load", "Bn_load", "opt_load", "writeback", "grad_offload")},
        "h2d_GBps": round(h2d_b / (per["h2d_ms"] / 1e3) / 1e9, 2) if per["h2d_ms"] else None,
        "d2h_GBps": round(d2h_b / (per["d2h_ms"] / 1e3) / 1e9, 2) if per["d2h_ms"] else None,
        "copy_engine_busy_s": {"h2d": round(per["h2d_ms"] / 1e3, 4), "d2h": round(per["d2h_ms"] / 1e3, 4)},
        "hidden_fraction": round(hidden, 4),
        "tokens_per_s": {"resident": round(T / t_res, 1), "offload": round(T / t_off, 1)},
        "spec_4W_no_overlap_prediction_s": round(p2r.predict_step_time(
            [gran // 18 * 4] * L, plan, h2d_b / (per["h2d_ms"] / 1e3) if per["h2d_ms"] else 50e9, t_nocopy), 4),
    }
    out["b200_overlap_prediction_s"] = round(overlap_prediction(p2r, out, L), 4)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
