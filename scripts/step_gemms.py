"""The twelve GEMMs of one C2 layer step exactly as the engine issues them
(layouts, epilogues, library-chosen split-K; csrc/engine/engine.cpp), timed with
CUDA events back to back (L2 warm, like consecutive launches in the step), next to
cuBLAS on the same operand shapes (plain bf16 / fp32 output, no fused epilogue).

  python scripts/step_gemms.py [--iters 30]
"""
import argparse
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_03888_b200 import _lib  # noqa: E402

T, d, f = 8192, 1024, 4096


def bf(*s):
    return torch.randn(*s, device="cuda").bfloat16()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--only", default=None, help="run just the GEMM of this name (profiling)")
    ap.add_argument("--variants", action="store_true", help="also time epilogue variants of the FFN1 shape")
    ap.add_argument("--split", type=int, default=None, help="force split_k on the dW GEMMs (measurement)")
    a = ap.parse_args()
    L = _lib.lib()
    x32 = torch.randn(T, d, device="cuda")
    a16, o16, b16, dy16, dx1_16 = bf(T, d), bf(T, d), bf(T, d), bf(T, d), bf(T, d)
    g16, hpre16, dh16 = bf(T, f), bf(T, f), bf(T, f)
    dqkv16 = bf(T, 3 * d)
    wqkv, wo, w1, w2 = bf(d, 3 * d), bf(d, d), bf(d, f), bf(f, d)
    b1, b2 = torch.randn(f, device="cuda"), torch.randn(d, device="cuda")
    out16 = torch.empty(T, f, device="cuda", dtype=torch.bfloat16)
    out16b = torch.empty(T, f, device="cuda", dtype=torch.bfloat16)
    out32 = torch.empty(T, max(f, 3 * d), device="cuda")
    gw = torch.zeros(f * d, device="cuda")
    db1 = torch.zeros(f, device="cuda")
    E = _lib
    # (name, m, n, k, A, lda, amn, B, ldb, bmn, epi, c, ldc, c2, ldc2, bias, aux, ldaux, split, bias_grad, cublas)
    cases = [
        ("QKV fwd", T, 3 * d, d, a16, d, 0, wqkv, 3 * d, 1, E.EPI_BF16, out16, 3 * d, None, 0, None, None, 0, 1, None,
         lambda: a16 @ wqkv),
        ("O fwd (+res)", T, d, d, o16, d, 0, wo, d, 1, E.EPI_F32, out32, d, None, 0, None, x32, d, 1, None,
         lambda: o16 @ wo),
        ("FFN1 fwd (+b,gelu)", T, f, d, b16, d, 0, w1, f, 1, E.EPI_BIAS_GELU, out16, f, out16b, f, b1, None, 0, 1, None,
         lambda: b16 @ w1),
        ("FFN1 shape, bf16", T, f, d, b16, d, 0, w1, f, 1, E.EPI_BF16, out16, f, None, 0, None, None, 0, 1, None,
         lambda: b16 @ w1),
        ("FFN1 shape, bf16+b", T, f, d, b16, d, 0, w1, f, 1, E.EPI_BF16, out16, f, None, 0, b1, None, 0, 1, None,
         lambda: b16 @ w1),
        ("FFN2 fwd (+b,res)", T, d, f, g16, f, 0, w2, d, 1, E.EPI_F32, out32, d, None, 0, b2, x32, d, 1, None,
         lambda: g16 @ w2),
        ("dW2", f, d, T, g16, f, 1, dy16, d, 1, E.EPI_ACC_F32, gw, d, None, 0, None, None, 0, 0, None,
         lambda: g16.T @ dy16),
        ("dH (gelu', db1)", T, f, d, dy16, d, 0, w2, d, 0, E.EPI_DGELU, out16, f, None, 0, None, hpre16, f, 1, db1,
         lambda: dy16 @ w2.T),
        ("dH shape, bf16", T, f, d, dy16, d, 0, w2, d, 0, E.EPI_BF16, out16, f, None, 0, None, None, 0, 1, None,
         lambda: dy16 @ w2.T),
        ("dH shape, no colsum", T, f, d, dy16, d, 0, w2, d, 0, E.EPI_DGELU, out16, f, None, 0, None, hpre16, f, 1,
         None, lambda: dy16 @ w2.T),
        ("dW1", d, f, T, b16, d, 1, dh16, f, 1, E.EPI_ACC_F32, gw, f, None, 0, None, None, 0, 0, None,
         lambda: b16.T @ dh16),
        ("dX1", T, d, f, dh16, f, 0, w1, f, 0, E.EPI_BF16, out16, d, None, 0, None, None, 0, 1, None,
         lambda: dh16 @ w1.T),
        ("dWo", d, d, T, o16, d, 1, dx1_16, d, 1, E.EPI_ACC_F32, gw, d, None, 0, None, None, 0, 0, None,
         lambda: o16.T @ dx1_16),
        ("dO", T, d, d, dx1_16, d, 0, wo, d, 0, E.EPI_BF16, out16, d, None, 0, None, None, 0, 1, None,
         lambda: dx1_16 @ wo.T),
        ("dWqkv", d, 3 * d, T, a16, d, 1, dqkv16, 3 * d, 1, E.EPI_ACC_F32, gw, 3 * d, None, 0, None, None, 0, 0, None,
         lambda: a16.T @ dqkv16),
        ("dXqkv", T, d, 3 * d, dqkv16, 3 * d, 0, wqkv, 3 * d, 0, E.EPI_BF16, out16, d, None, 0, None, None, 0, 1, None,
         lambda: dqkv16 @ wqkv.T),
    ]
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot_us = tot_cb = tot_f = 0.0
    print(f"{'gemm':20s} {'m':>6s} {'n':>5s} {'k':>5s}   p2r us  TFLOP/s | cuBLAS us TFLOP/s")
    for (name, m, n, k, A, lda, amn, B, ldb, bmn, epi, c, ldc, c2, ldc2, bias, aux, ldaux, split, bgrad, cb) in cases:
        if a.only is not None and name != a.only:
            continue
        if a.only is None and "shape" in name and not a.variants:
            continue
        args = _lib.GemmArgs(m=m, n=n, k=k, a=A.data_ptr(), lda=lda, a_mn_major=amn, b=B.data_ptr(), ldb=ldb,
                             b_mn_major=bmn, epi=epi, c=c.data_ptr(), ldc=ldc,
                             c2=c2.data_ptr() if c2 is not None else None, ldc2=ldc2,
                             bias=bias.data_ptr() if bias is not None else None,
                             aux=aux.data_ptr() if aux is not None else None, ldaux=ldaux,
                             split_k=a.split if (a.split is not None and name.startswith("dW")) else split,
                             bias_grad=bgrad.data_ptr() if bgrad is not None else None)
        ws = torch.empty(max(1, L.p2r_gemm_workspace_bytes(ctypes.byref(args)) // 4), device="cuda")
        _lib.check(L.p2r_set_workspace(ws.data_ptr(), ws.numel() * 4))
        for _ in range(3):
            _lib.check(L.p2r_gemm(ctypes.byref(args), s))
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            _lib.check(L.p2r_gemm(ctypes.byref(args), s))
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.iters * 1e3
        for _ in range(3):
            cb()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            cb()
        e1.record()
        torch.cuda.synchronize()
        ucb = e0.elapsed_time(e1) / a.iters * 1e3
        fl = 2.0 * m * n * k
        tot_us += us
        tot_cb += ucb
        tot_f += fl
        print(f"{name:20s} {m:6d} {n:5d} {k:5d} {us:8.1f} {fl / us / 1e6:8.1f} | {ucb:8.1f} {fl / ucb / 1e6:8.1f}")
    print(f"{'layer total':20s} {'':18s} {tot_us:8.1f} {tot_f / tot_us / 1e6:8.1f} | {tot_cb:8.1f} "
          f"{tot_f / tot_cb / 1e6:8.1f}")


if __name__ == "__main__":
    main()
