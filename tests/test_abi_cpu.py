"""CPU: the C-ABI library loads, exports every symbol include/*.h declares, and
its host-only entry points (init RNG, count_params, LR schedule, capacity)
agree with the reference. No device compute here."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2110_03888_b200", "libp2r.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libp2r_ref.so")

need_lib = pytest.mark.skipif(not os.path.exists(LIB), reason="libp2r.so not built (make)")


def declared_symbols():
    syms = set()
    for h in ("p2r_cuda.h", "p2r_engine.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        syms |= set(re.findall(r"\b(p2r_[a-z0-9_]+)\s*\(", src))
    return syms


@need_lib
def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(LIB)
    missing = [s for s in sorted(declared_symbols()) if not hasattr(L, s)]
    assert not missing, missing
    assert len(declared_symbols()) >= 40


@need_lib
def test_version_and_errors():
    import paper_2110_03888_b200 as p2r
    L = p2r.lib()
    assert b"sm_100a" in L.p2r_version()
    args = p2r._lib.GemmArgs(m=-1, n=1, k=1)
    st = L.p2r_gemm(ctypes.byref(args), None)
    assert st == p2r._lib.P2R_EINVAL
    assert b"negative dimension" in L.p2r_last_error()


@need_lib
def test_count_params_and_lr_match_reference_golden():
    import paper_2110_03888_b200 as p2r
    d = dict(np.load(os.path.join(ROOT, "tests", "golden", "primitives.npz")))
    pseudo = p2r.Config(d_model=1024, d_ff=16384, n_layers_graph=36, n_layers_params=1, n_heads=16, vocab_size=50000, seq_len=512)
    assert p2r.count_params(pseudo) == tuple(d["count.pseudo"])
    c1 = p2r.Config(d_model=256, d_ff=1024, n_layers_graph=4, n_layers_params=1, n_heads=4, vocab_size=260, seq_len=128, n_experts=4)
    assert p2r.count_params(c1) == tuple(d["count.c1"]) == (99840, 2366464, 2466304)
    lrs = np.array([p2r.lr_at(2e-4, 0.1, 100, int(s)) for s in d["lr.steps"]], np.float32)
    assert np.array_equal(lrs, d["lr.values"])
    with pytest.raises(p2r.P2RInvalidArgument, match="divisible by n_heads"):
        p2r.count_params(p2r.Config(d_model=250, n_heads=4))


@need_lib
def test_capacity_formula():
    import paper_2110_03888_b200 as p2r
    from paper_2110_03888_b200.model import _declare_extra
    L = _declare_extra()
    # model.cpp:308-309: ceil(double(cf) * T / gs)
    assert L.p2r_moe_capacity(1.25, 1024, 4, 1) == 320
    assert L.p2r_moe_capacity(1.0, 4, 4, 1) == 1
    assert L.p2r_moe_capacity(1.0, 257, 8, 2) == 65


@need_lib
@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")
def test_init_rng_bit_exact_vs_reference():
    """The engine's host init (same std::mt19937_64 + normal_distribution<float>)
    reproduces the reference's initial weights bit for bit."""
    from oracle import ref
    from paper_2110_03888_b200._lib import lib
    L = lib()
    L.p2r_init_normal_host.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int64, ctypes.c_void_p]
    L.p2r_init_normal_host.restype = None
    cfg = ref.Config(d_model=64, d_ff=128, n_layers_graph=3, n_layers_params=1, n_heads=2,
                     vocab_size=260, seq_len=16, n_experts=4)
    r = ref.RefModel(cfg, 1234)
    params = r.params()
    for n in ("embed.tok", "embed.pos", "layer.0.attn.wq", "layer.0.moe.gate", "layer.0.moe.expert.3.w2"):
        out = np.empty(params[n].size, np.float32)
        L.p2r_init_normal_host(1234, n.encode(), out.size, out.ctypes.data_as(ctypes.c_void_p))
        assert np.array_equal(out.reshape(params[n].shape), params[n]), n
