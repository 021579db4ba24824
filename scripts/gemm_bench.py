"""Quick p2r_gemm throughput probe (CUDA events) on the C2 training-step GEMM shapes."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2110_03888_b200 import _lib  # noqa: E402


def run(m, n, k, amn=0, bmn=0, epi=_lib.EPI_BF16, split=1, iters=20, bias_grad=False):
    dev = torch.device("cuda")
    A = torch.randn(k, m, device=dev).bfloat16() if amn else torch.randn(m, k, device=dev).bfloat16()
    B = torch.randn(k, n, device=dev).bfloat16() if bmn else torch.randn(n, k, device=dev).bfloat16()
    C = torch.zeros(m, n, device=dev, dtype=torch.float32)
    C2 = torch.zeros(m, n, device=dev, dtype=torch.bfloat16)
    args = _lib.GemmArgs(m=m, n=n, k=k, a=A.data_ptr(), lda=A.shape[1], a_mn_major=amn,
                         b=B.data_ptr(), ldb=B.shape[1], b_mn_major=bmn, epi=epi,
                         c=C.data_ptr(), ldc=n, c2=C2.data_ptr(), ldc2=n, split_k=split)
    if epi in (_lib.EPI_BF16, _lib.EPI_BIAS_GELU):
        args.c = C2.data_ptr()
    if epi == _lib.EPI_BIAS_GELU:
        args.c2 = C.data_ptr()  # any bf16-sized buffer works (fp32 is 2x larger)
    if epi == _lib.EPI_DGELU:
        AUX = torch.randn(m, n, device=dev).bfloat16()
        args.c = C2.data_ptr()
        args.aux = AUX.data_ptr()
        args.ldaux = n
    if bias_grad:
        DB = torch.zeros(n, device=dev)
        args.bias_grad = DB.data_ptr()
    ws = torch.empty(max(1, _lib.lib().p2r_gemm_workspace_bytes(ctypes.byref(args)) // 4), device=dev)
    _lib.check(_lib.lib().p2r_set_workspace(ws.data_ptr(), ws.numel() * 4))
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        _lib.check(_lib.lib().p2r_gemm(ctypes.byref(args), s))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        _lib.check(_lib.lib().p2r_gemm(ctypes.byref(args), s))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tf = 2.0 * m * n * k / ms / 1e9
    # torch (cuBLAS) for context
    Af = A.T if amn else A
    Bf = B if bmn else B.T
    for _ in range(3):
        torch.matmul(Af, Bf)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        torch.matmul(Af, Bf)
    e1.record()
    torch.cuda.synchronize()
    ms_t = e0.elapsed_time(e1) / iters
    print(f"m={m:6d} n={n:5d} k={k:5d} amn={amn} bmn={bmn} epi={epi} split={split}{' +db' if bias_grad else ''}: "
          f"{ms*1e3:8.1f} us {tf:7.1f} TFLOP/s   (cuBLAS {ms_t*1e3:8.1f} us {2.0*m*n*k/ms_t/1e9:7.1f})")


if __name__ == "__main__":
    T, d, f = 8192, 1024, 4096
    run(T, 3 * d, d)                       # QKV
    run(T, d, d, epi=_lib.EPI_F32)         # O proj (+resid)
    run(T, f, d, epi=_lib.EPI_BIAS_GELU)   # FFN1
    run(T, f, d)                           # FFN1 shape, plain bf16 epilogue
    run(T, f, d, epi=_lib.EPI_DGELU)       # dH = dY W2^T * gelu'(h)
    run(T, d, f, epi=_lib.EPI_F32)         # FFN2
    run(T, d, 3 * d, epi=_lib.EPI_F32)     # dX of QKV
    run(d, 3 * d, T, amn=1, bmn=1, epi=_lib.EPI_ACC_F32, split=1)  # dWqkv
    run(d, 3 * d, T, amn=1, bmn=1, epi=_lib.EPI_ACC_F32, split=2)
    run(d, d, T, amn=1, bmn=1, epi=_lib.EPI_ACC_F32, split=4)
    run(d, f, T, amn=1, bmn=1, epi=_lib.EPI_ACC_F32, split=2)
    run(8192, 8192, 8192)
