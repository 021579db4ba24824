"""Run a single p2r_gemm shape a few times (for ncu captures)."""
import sys
sys.path.insert(0, ".")
from scripts.gemm_bench import run
from paper_2110_03888_b200 import _lib
shape = sys.argv[1] if len(sys.argv) > 1 else "ffn1"
T, d, f = 8192, 1024, 4096
if shape == "ffn1":
    run(T, f, d, epi=_lib.EPI_BIAS_GELU, iters=3)
elif shape == "dgelu":
    run(T, f, d, epi=_lib.EPI_DGELU, iters=3)
elif shape == "qkv":
    run(T, 3 * d, d, iters=3)
elif shape == "dw":
    run(d, 3 * d, T, amn=1, bmn=1, epi=_lib.EPI_ACC_F32, iters=3)
elif shape == "big":
    run(8192, 8192, 8192, iters=3)
