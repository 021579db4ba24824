"""ORACLE / TEST INFRASTRUCTURE ONLY — where the bf16-in design's gradient error
comes from. Runs oracle/bf16_emulation.py (the fp32 model with bf16 rounding at
exactly the GPU path's rounding points) with all points, with one point at a time
raised to fp32, and with groups of points raised, and prints the worst per-tensor
gradient rel-L2 against the fp32 model (points=()) on the same inputs.

  python -m oracle.precision_floor [--d 256 --layers 3 --params 3 --seq 128 --batch 8]

Result recorded in DESIGN.md §4: at random init the attention Q/K projection
gradients of unshared layers sit at ~1.0-1.4 % and no single rounding point
(in particular not the dQ/dK -> dW_qkv path) moves them below ~1.0 %.
Parameters come from the compiled reference's init (oracle/_ref)."""
from __future__ import annotations

import argparse

import numpy as np

from . import bf16_emulation as BE
from . import p2r_oracle as O
from . import ref


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--params", type=int, default=3)
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--batch", type=int, default=8)
    a = ap.parse_args()
    cfgd = dict(d_model=a.d, d_ff=4 * a.d, n_layers_graph=a.layers, n_layers_params=a.params,
                n_heads=a.d // 64, vocab_size=260, seq_len=a.seq)
    cfg = O.Config(**cfgd)
    p0 = ref.RefModel(ref.Config(**cfgd), 1234).params()
    rng = np.random.default_rng(7)
    tok = rng.integers(0, 256, (a.batch, a.seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    tok, tgt, mask = tok.ravel(), tgt.ravel(), mask.ravel()
    denom = float(mask.sum())
    pts_all = tuple(p for p in BE.ALL_POINTS if p not in ("ye16", "dye16", "dxe16"))  # dense stack
    _, g0 = BE.loss_and_grads(cfg, p0, tok, tgt, mask, a.batch, denom, points=())

    def worst(pts):
        _, g = BE.loss_and_grads(cfg, p0, tok, tgt, mask, a.batch, denom, points=pts)
        rows = sorted(((float(np.linalg.norm(g[n].astype(np.float64) - g0[n]) / np.linalg.norm(g0[n])), n)
                       for n in g0 if np.linalg.norm(g0[n]) > 0), reverse=True)
        return rows[0]

    print(f"config {cfgd} batch {a.batch}")
    e, n = worst(pts_all)
    print(f"{'all rounding points':34s} worst {e:.4f} {n}")
    for p in pts_all:
        e, n = worst(tuple(x for x in pts_all if x != p))
        print(f"{'all but ' + p:34s} worst {e:.4f} {n}")
    fwd = ("w16", "a16", "qkv16", "p16", "o16", "b16", "gd16", "g16", "h16")
    for tag, pts in (("forward points only", fwd),
                     ("backward points only", tuple(x for x in pts_all if x not in fwd)),
                     ("weights (w16) only", ("w16",)),
                     ("all but a16,qkv16,o16,w16", tuple(x for x in pts_all if x not in ("a16", "qkv16", "o16", "w16")))):
        e, n = worst(pts)
        print(f"{tag:34s} worst {e:.4f} {n}")


if __name__ == "__main__":
    main()
