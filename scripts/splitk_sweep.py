"""dW (C += A^T B, K = tokens) split-K sweep over the C2 step's shapes:
python scripts/splitk_sweep.py  (set P2R_GEMM_SERIAL=0 for the partials+reduce path)."""
import os
import sys

sys.path.insert(0, ".")
from scripts.gemm_bench import run  # noqa: E402
from paper_2110_03888_b200 import _lib  # noqa: E402

T, d, f = 8192, 1024, 4096
print("serial" if os.environ.get("P2R_GEMM_SERIAL", "1") != "0" else "partials+reduce")
for m, n in ((d, 3 * d), (d, d), (d, f), (f, d)):
    for split in ((0,) if os.environ.get("AUTO_ONLY") else (0, 1, 2, 3, 4)):
        run(m, n, T, amn=1, bmn=1, epi=_lib.EPI_ACC_F32, split=split)
