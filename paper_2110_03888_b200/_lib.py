"""ctypes binding of the C-ABI declared in include/p2r_cuda.h and include/p2r_engine.h.

The product path is libp2r.so (sm_100a kernels + C++ host engine). There is no
Python or CPU fallback: if the library is missing, importing raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# P2R_LIB selects another build of the same library (diagnostic ablation builds)
LIB_PATH = os.environ.get("P2R_LIB") or os.path.join(_HERE, "libp2r.so")

P2R_OK, P2R_EINVAL, P2R_ERANGE, P2R_ELOGIC, P2R_ERUNTIME, P2R_ECUDA, P2R_ENCCL = range(7)

EPI_BF16, EPI_F32, EPI_ACC_F32, EPI_BIAS_GELU, EPI_DGELU, EPI_F32_BF16 = range(6)
GROUP_NONE, GROUP_M, GROUP_K = range(3)


class P2RError(RuntimeError):
    pass


class P2RInvalidArgument(P2RError, ValueError):
    """std::invalid_argument in the reference."""


class P2ROutOfRange(P2RError, IndexError):
    """std::out_of_range in the reference."""


class P2RLogicError(P2RError):
    """std::logic_error in the reference."""


_EXC = {
    P2R_EINVAL: P2RInvalidArgument,
    P2R_ERANGE: P2ROutOfRange,
    P2R_ELOGIC: P2RLogicError,
}


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int), ("n", ctypes.c_int), ("k", ctypes.c_int),
        ("a", ctypes.c_void_p), ("lda", ctypes.c_int), ("a_mn_major", ctypes.c_int),
        ("b", ctypes.c_void_p), ("ldb", ctypes.c_int), ("b_mn_major", ctypes.c_int),
        ("epi", ctypes.c_int),
        ("c", ctypes.c_void_p), ("ldc", ctypes.c_int),
        ("c2", ctypes.c_void_p), ("ldc2", ctypes.c_int),
        ("bias", ctypes.c_void_p),
        ("aux", ctypes.c_void_p), ("ldaux", ctypes.c_int),
        ("group_mode", ctypes.c_int), ("groups", ctypes.c_int), ("seg_rows", ctypes.c_int),
        ("counts", ctypes.c_void_p),
        ("split_k", ctypes.c_int),
        ("cta_group", ctypes.c_int),
        ("bias_grad", ctypes.c_void_p),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise P2RError(
                f"{LIB_PATH} not built: run `make` (or __graft_entry__.build()); "
                "there is no CPU fallback")
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    L.p2r_last_error.restype = ctypes.c_char_p
    L.p2r_version.restype = ctypes.c_char_p
    L.p2r_launch_count.restype = ctypes.c_uint64
    L.p2r_gemm.argtypes = [ctypes.POINTER(GemmArgs), ctypes.c_void_p]
    L.p2r_gemm.restype = ctypes.c_int
    L.p2r_gemm_workspace_bytes.argtypes = [ctypes.POINTER(GemmArgs)]
    L.p2r_gemm_workspace_bytes.restype = ctypes.c_size_t
    L.p2r_set_workspace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    L.p2r_set_workspace.restype = ctypes.c_int
    for name in ("p2r_embed_bwd_workspace", "p2r_colsum_workspace", "p2r_layernorm_bwd_workspace",
                 "p2r_cross_entropy_workspace"):
        getattr(L, name).restype = ctypes.c_size_t
    for name, argtypes in _EXTRA_SIGNATURES.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int


# Filled in by the modules that bind further entry points.
_EXTRA_SIGNATURES: dict = {}


def check(status: int) -> None:
    if status != P2R_OK:
        msg = lib().p2r_last_error().decode()
        raise _EXC.get(status, P2RError)(msg)


def launch_count() -> int:
    return int(lib().p2r_launch_count())
