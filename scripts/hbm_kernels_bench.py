"""Achieved HBM GB/s of the routing / dispatch / combine and delink kernels (north star:
"achieved HBM GB/s against about 8 TB/s for the elementwise, routing and delink kernels").

Shapes: MoE kernels at the C4 per-rank shape (T = 8192 tokens, d = 2048,
E = 64 experts, top-1, capacity factor 1.25 -> capacity 160, 256-row expert segments);
delink at C3 (one shared layer of d = 1024, d_ff = 4096 -> 12.6 M params per GPU, its
p32 / m / v fp32 buffers and bf16 operand broadcast into L = 24 layers). Each launch is
timed alone with CUDA events after an L2 flush (256 MB write), median of 20.
Algorithmic bytes per launch are the §8(d) figures, written next to each row.

  python scripts/hbm_kernels_bench.py [--out profiles/r01_hbm_kernels.json]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2110_03888_b200 import _lib
    L = _lib.lib()
    st = torch.cuda.current_stream()
    S = ctypes.c_void_p(st.cuda_stream)
    P = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
    dev = "cuda"
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 7672.0}
    hbm = float(peaks["hbm_gbs"])

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.iters):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return float(np.median(ts))

    rows = []

    def record(name, us, nbytes, note):
        gbs = nbytes / (us * 1e-6) / 1e9
        rows.append({"kernel": name, "us": round(us, 2), "algorithmic_bytes": int(nbytes), "gbs": round(gbs, 1),
                     "frac_hbm": round(gbs / hbm, 3), "bytes": note})
        print(f"{name:28s} {us:9.2f} us  {nbytes / 1e6:9.2f} MB  {gbs:8.1f} GB/s  ({gbs / hbm:.2f} of {hbm:.0f})")

    def ck(s):
        _lib.check(s)

    # ---------------- MoE at the C4 per-rank shape ----------------
    T, d, E, k = 8192, 2048, 64, 1
    cap = L.p2r_moe_capacity(ctypes.c_float(1.25), T, E, k)
    seg = max(128, (min(cap, T) + 127) // 128 * 128)
    ES = E * seg
    g = torch.Generator(device=dev).manual_seed(0)
    b32 = torch.randn(T, d, device=dev, generator=g)
    b16 = b32.bfloat16()
    gate = torch.randn(d, E, device=dev, generator=g) * 0.02
    logits = torch.empty(T, E, device=dev)
    sel = torch.empty(T * k, dtype=torch.int32, device=dev)
    surv = torch.empty(T * k, dtype=torch.uint8, device=dev)
    pos = torch.empty(T * k, dtype=torch.int32, device=dev)
    raw = torch.empty(E, dtype=torch.int32, device=dev)
    counts = torch.empty(E, dtype=torch.int32, device=dev)
    rows_pad = torch.empty(ES, dtype=torch.int32, device=dev)
    slots_pad = torch.empty(ES, dtype=torch.int32, device=dev)
    dropped = torch.empty(1, dtype=torch.int32, device=dev)
    w = torch.empty(T * k, device=dev)
    xe16 = torch.zeros(ES, d, dtype=torch.bfloat16, device=dev)
    ye32 = torch.randn(ES, d, device=dev, generator=g)
    resid = torch.randn(T, d, device=dev, generator=g)
    out = torch.empty(T, d, device=dev)
    dout = torch.randn(T, d, device=dev, generator=g)
    dw = torch.empty(T * k, device=dev)
    dxe = torch.randn(ES, d, device=dev, generator=g)
    db = torch.empty(T, d, device=dev)

    gate_fn = lambda: ck(L.p2r_moe_gate_logits(P(b32), P(gate), T, d, E, P(logits), S))  # noqa: E731
    gate_fn()
    route_fn = lambda: ck(L.p2r_moe_route(P(logits), T, E, k, cap, seg, P(sel), P(surv), P(pos), P(raw),  # noqa: E731
                                          P(counts), P(rows_pad), P(slots_pad), P(dropped), S))
    route_fn()
    ck(L.p2r_moe_combine_weights(P(logits), T, E, k, P(sel), P(surv), P(w), S))
    torch.cuda.synchronize()
    admitted = int(counts.sum())
    record("moe_gate_logits (fp32)", timed(gate_fn), 4 * T * d + 4 * d * E + 4 * T * E,
           "4Td (b) + 4dE (gate) + 4TE (logits)")
    record("moe_route", timed(route_fn), 4 * T * E + 13 * T * k + 8 * ES,
           "4TE logits in; 13Tk (sel, surv, pos, w-slot) + 8·E·seg (rows/slots) out")
    record("moe_combine_weights", timed(lambda: ck(L.p2r_moe_combine_weights(
        P(logits), T, E, k, P(sel), P(surv), P(w), S))), 4 * T * E + 9 * T * k, "4TE + 9Tk")
    record("moe_dispatch (bf16)", timed(lambda: ck(L.p2r_moe_dispatch(
        P(b16), 1, d, E, seg, P(rows_pad), P(slots_pad), P(counts), None, k, P(xe16), 0, S))),
        2 * 2 * admitted * d, f"2·admitted·d·2 (admitted rows {admitted})")
    record("moe_combine (+resid)", timed(lambda: ck(L.p2r_moe_combine(
        P(ye32), T, d, k, seg, P(sel), P(pos), P(w), P(resid), P(out), S))), 4 * admitted * d + 8 * T * d,
        "4·admitted·d (ye) + 4Td (resid) + 4Td (out)")
    record("moe_combine_bwd_weights", timed(lambda: ck(L.p2r_moe_combine_bwd_weights(
        P(dout), P(ye32), T, d, k, seg, P(sel), P(pos), P(dw), S))), 4 * T * d + 4 * admitted * d,
        "4Td (dout) + 4·admitted·d (ye)")
    record("moe_dispatch dy (fp32->bf16)", timed(lambda: ck(L.p2r_moe_dispatch(
        P(dout), 0, d, E, seg, P(rows_pad), P(slots_pad), P(counts), P(w), k, P(xe16), 0, S))),
        (4 + 2) * admitted * d, "4·admitted·d in + 2·admitted·d out")
    record("moe_dispatch_bwd", timed(lambda: ck(L.p2r_moe_dispatch_bwd(
        P(dxe), T, d, k, seg, P(sel), P(pos), None, P(gate), E, P(db), 0, S))), 4 * admitted * d + 4 * T * d,
        "4·admitted·d (dxe) + 4Td (db)")
    del ye32, dxe, xe16, b32, b16, resid, out, dout, db
    torch.cuda.empty_cache()
    # C3 per-rank gate: d = 1024, E = 8 (one expert per GPU, every rank scores all 8)
    T3, d3, E3 = 8192, 1024, 8
    b3 = torch.randn(T3, d3, device=dev, generator=g)
    gate3 = torch.randn(d3, E3, device=dev, generator=g) * 0.02
    lg3 = torch.empty(T3, E3, device=dev)
    record("moe_gate_logits C3 (E=8)", timed(lambda: ck(L.p2r_moe_gate_logits(P(b3), P(gate3), T3, d3, E3, P(lg3), S))),
           4 * T3 * d3 + 4 * d3 * E3 + 4 * T3 * E3, "4Td + 4dE + 4TE")
    del b3

    # ---------------- delink at C3 (one shared layer -> 24) ----------------
    Ld, dm, dff = 24, 1024, 4096
    n = 4 * dm * dm + 2 * dm * dff + dff + dm + 4 * dm  # one C3 layer granule: QKV+O, FFN, biases, 2 LN
    tot = 0.0
    nb = 0
    for esize in (4, 4, 4, 2):  # p32, m, v, bf16 operand
        src = torch.empty(n * esize, dtype=torch.uint8, device=dev).random_(0, 255)
        dst = torch.empty(Ld, n * esize, dtype=torch.uint8, device=dev)
        us = timed(lambda: ck(L.p2r_delink_broadcast(P(src), P(dst), ctypes.c_size_t(n * esize),
                                                     ctypes.c_size_t(n * esize), Ld, S)))
        assert bool((dst[Ld - 1] == src).all())
        tot += us
        nb += (1 + Ld) * n * esize
        del src, dst
        torch.cuda.empty_cache()
    record("delink_broadcast (C3 granule)", tot, nb, "(1 + L)·granule bytes, p32 + m + v + bf16 (14 B/param)")

    res = {"shapes": {"moe": f"T={T} d={d} E={E} k={k} cap={cap} seg={seg} admitted={admitted}",
                      "delink": f"L={Ld} granule {n} params x 14 B"},
           "hbm_peak_gbs": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy read+write)",
           "timing": "CUDA events per launch after a 256 MB L2 flush, median of %d" % args.iters, "kernels": rows}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
