"""Ablation builds of the attention backward kernels (diagnostics only).

Writes modified copies of csrc/attention_bwd_tc.cu to build/exp/, links each
into build/exp/libp2r_<variant>.so, so scripts/attn_bench.py can time them via
P2R_LIB=<path>:
  nomma  - no tcgen05.mma issued (commits still flow): softmax/TMA-bound time
  nosm   - softmax warps skip TMEM loads and math (stores/barriers kept)
  nodq / nokv - launch only the dK/dV (resp. dQ) kernel (compose: nodq+nomma, ...)
  trace  - P2R_ATTN_TRACE: clock64 timeline of one dQ CTA (scripts/attn_trace.py)
"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2110_03888_b200/csrc/attention_bwd_tc.cu")
OUT = os.path.join(ROOT, "build/exp")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def variant(name, text):
    if "+" in name:  # composable: e.g. trace+nosm
        for part in name.split("+"):
            text = variant(part, text)
        return text
    if name == "nomma":
        text = text.replace("umma_bf16(", "if (false) umma_bf16(").replace("umma_bf16_warp(", "if (false) umma_bf16_warp(")
    elif name == "nosm":
        text = re.sub(r"ld32x2\((tmem|tS)[^;]*\);", r"{ for (int z_ = 0; z_ < 32; ++z_) { s[z_] = 0.f; dp[z_] = 0.f; } }", text)
        text = re.sub(r"\? ex2_approx\(", "? (", text)
    elif name == "nodq":  # time the dK/dV kernel alone (dsum left from an earlier full run)
        text = text.replace('P2R_LAUNCH_K("attention bwd dq (tcgen05, 2 tiles, persistent)"',
                            'if (false) P2R_LAUNCH_K("attention bwd dq (tcgen05, 2 tiles, persistent)"')
    elif name == "nokv":  # time the dQ kernel alone
        text = text.replace('P2R_LAUNCH_K("attention bwd dkdv (tcgen05, 2 tiles, persistent)"',
                            'if (false) P2R_LAUNCH_K("attention bwd dkdv (tcgen05, 2 tiles, persistent)"')
    elif name.startswith("fma"):  # fwd: fmaN = N of 8 chunks' exponentials on the FMA pipe
        text = "#define P2R_ATTN_FMA_CHUNKS " + name[3:] + "\n" + text
    elif name == "trace":
        text = "#define P2R_ATTN_TRACE 1\n" + text
    return text


def main(names, src=SRC):
    """fwd variants: prefix the name with "fwd:" (patches csrc/attention_tc.cu)."""
    os.makedirs(OUT, exist_ok=True)
    stem = os.path.basename(src)[:-3]
    base = open(src).read().replace('"../../include/p2r_cuda.h"', '"p2r_cuda.h"')
    others = [o for o in glob.glob(os.path.join(ROOT, "build/*.o")) if not o.endswith(stem + ".o")]
    eng = glob.glob(os.path.join(ROOT, "build/engine/*.o"))
    for n in names:
        cu = os.path.join(OUT, f"{stem}_{n.replace('+', '_')}.cu")
        open(cu, "w").write(variant(n, base))
        obj = cu[:-3].replace("+", "_") + ".o"
        subprocess.check_call(["nvcc", *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
                               "-I" + os.path.join(ROOT, "paper_2110_03888_b200/csrc"), "--expt-relaxed-constexpr",
                               "-c", cu, "-o", obj])
        subprocess.check_call(["nvcc", *ARCH, "-shared", "-o", os.path.join(OUT, f"libp2r_{'' if stem.startswith('attention_bwd') else stem + '_'}{n.replace('+', '_')}.so"), *others, obj, *eng,
                               "-cudart", "static"])
        print("built", n)


if __name__ == "__main__":
    args = sys.argv[1:] or ["nomma", "nosm"]
    fwd = [a[4:] for a in args if a.startswith("fwd:")]
    bwd = [a for a in args if not a.startswith("fwd:")]
    if bwd:
        main(bwd)
    if fwd:
        main(fwd, os.path.join(ROOT, "paper_2110_03888_b200/csrc/attention_tc.cu"))
