"""Ablation builds of the GEMM epilogue (diagnostics only).

Writes modified copies of csrc/gemm_sm100.cu to build/exp/ and links each into
build/exp/libp2r_gemm_<variant>.so; time them with P2R_LIB=<path> scripts/gemm_bench.py.
  noepi   - epilogue warps drain TMEM and release it, nothing else (mainloop bound)
  nostage - no shared-memory transpose: values are taken straight from the TMEM
            registers (wrong placement, same global traffic and math)
  trace   - clock64 per-tile timeline of CTA 0 (producer / MMA / epilogue warp 4),
            dumped over the start of C (scripts/gemm_trace.py)
  span    - %globaltimer at entry / after setup / at exit for every CTA, written to
            C rows 1.. (scripts/gemm_trace.py --span)
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2110_03888_b200/csrc/gemm_sm100.cu")
OUT = os.path.join(ROOT, "build/exp")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sub(text, a, b):
    assert a in text, a
    return text.replace(a, b)


def variant(name, text):
    if name == "noepi":
        text = sub(text, "if (nrows <= 0 || col0 >= p.n) continue;  // warp-uniform", "continue;")
    elif name == "nogelu":  # GELU / GELU' replaced by identity (same loads and stores)
        text = sub(text, "pack4_bf16(gelu_f(pre.x), gelu_f(pre.y), gelu_f(pre.z), gelu_f(pre.w));\n  } else if constexpr",
                   "pack4_bf16(pre.x, pre.y, pre.z, pre.w);\n  } else if constexpr")
        text = sub(text, """        pack4_bf16(v.x * gelu_grad_f(pre.x), v.y * gelu_grad_f(pre.y), v.z * gelu_grad_f(pre.z),
                   v.w * gelu_grad_f(pre.w));
  }
}""", """        pack4_bf16(v.x * pre.x, v.y * pre.y, v.z * pre.z, v.w * pre.w);
  }
}""")
    elif name == "noc2":  # BIAS_GELU without the pre-activation store
        text = sub(text, """    const float4 pre = make_float4(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.c2) + row * p.ldc2 + col) =
        pack4_bf16(pre.x, pre.y, pre.z, pre.w);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) =
        pack4_bf16(gelu_f(""", """    const float4 pre = make_float4(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) =
        pack4_bf16(gelu_f(""")
    elif name == "nostage":
        text = sub(text, """        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(stg + lane * 32 + ((q ^ (lane & 7)) << 2)) =
              make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                          __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));""", "        for (int q = 0; q < 0; ++q) {}")
        text = sub(text, """            const float4 v = *reinterpret_cast<const float4*>(stg + rr * 32 + ((cg ^ (rr & 7)) << 2));
            epi_store_fast<EPI>""", """            const float4 v = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                         __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
            epi_store_fast<EPI>""")
    elif name == "trace":
        text = sub(text, """  const uint32_t tmem_base = *tmem_slot;
""", """  const uint32_t tmem_base = *tmem_slot;
  __shared__ long long s_tr[128];
  const bool trc = blockIdx.x == 0;
#define TRG(slot) do { if (trc && (slot) < 128) s_tr[(slot)] = clock64(); } while (0)
  if (threadIdx.x == 0) TRG(0);
  int tr_tile = 0;
""")
        # producer: first empty wait of each tile + last load issued
        text = sub(text, """        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          mbar_wait(empty_bar + stage, phase ^ 1);""", """        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          mbar_wait(empty_bar + stage, phase ^ 1);
          if (kb == T.kb0) TRG(8 + 8 * tr_tile);
          if (kb == T.kb1 - 1) TRG(8 + 8 * tr_tile + 1);""")
        text = sub(text, """          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {""", """          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        ++tr_tile;
      }
    }
  } else if (warp == 1) {""")
        text = sub(text, """        mbar_wait(tempty_bar + acc, acc_phase ^ 1);""", """        mbar_wait(tempty_bar + acc, acc_phase ^ 1);
        TRG(8 + 8 * tr_tile + 2);""")
        text = sub(text, """        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {""", """        TRG(8 + 8 * tr_tile + 3);
        ++tr_tile;
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {""")
        text = sub(text, """      mbar_wait(tfull_bar + acc, acc_phase);""", """      mbar_wait(tfull_bar + acc, acc_phase);
      if (warp == 4 && lane == 0) TRG(8 + 8 * tr_tile + 4);""")
        text = sub(text, """      tc_fence_before();
      if constexpr (CG == 2) {
        __syncwarp();""", """      if (warp == 4 && lane == 0) TRG(8 + 8 * tr_tile + 5);
      if (warp == 11 && lane == 0) TRG(8 + 8 * tr_tile + 6);
      ++tr_tile;
      tc_fence_before();
      if constexpr (CG == 2) {
        __syncwarp();""")
        text = sub(text, """    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}""", """    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
  if (trc && threadIdx.x == 0) {
    s_tr[1] = clock64();
    for (int i = 0; i < 128; ++i) reinterpret_cast<long long*>(p.c)[i] = s_tr[i];
  }
}""")
    elif name == "trace1":  # the trace timeline of CTA 1 (the pair's second CTA)
        text = variant("trace", text)
        text = sub(text, "const bool trc = blockIdx.x == 0;", "const bool trc = blockIdx.x == 1;")
    elif name == "span":
        text = sub(text, """  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
""", """  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long g_t0 = 0, g_t1 = 0, g_t2 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_t0));
""")
        text = sub(text, """  const uint32_t tmem_base = *tmem_slot;
""", """  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_t1));
""")
        text = sub(text, """    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}""", """    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
  if (threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_t2));
    unsigned long long* o = reinterpret_cast<unsigned long long*>(p.c) + 1024 + 4 * blockIdx.x;
    o[0] = g_t0;
    o[1] = g_t1;
    o[2] = g_t2;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    o[3] = smid;
  }
}""")
    return text


def main(names):
    os.makedirs(OUT, exist_ok=True)
    base = open(SRC).read().replace('"../../include/p2r_cuda.h"', '"p2r_cuda.h"')
    others = [o for o in glob.glob(os.path.join(ROOT, "build/*.o")) if not o.endswith("gemm_sm100.o")]
    eng = glob.glob(os.path.join(ROOT, "build/engine/*.o"))
    for n in names:
        cu = os.path.join(OUT, f"gemm_sm100_{n}.cu")
        open(cu, "w").write(variant(n, base))
        obj = cu[:-3] + ".o"
        subprocess.check_call(["nvcc", *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
                               "-I" + os.path.join(ROOT, "paper_2110_03888_b200/csrc"), "--expt-relaxed-constexpr",
                               "-c", cu, "-o", obj])
        subprocess.check_call(["nvcc", *ARCH, "-shared", "-o", os.path.join(OUT, f"libp2r_gemm_{n}.so"), *others, obj,
                               *eng, "-cudart", "static"])
        print("built", n)


if __name__ == "__main__":
    main(sys.argv[1:] or ["noepi", "nostage"])
