"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes driver of the compiled reference.

Loads oracle/_ref/libp2r_ref.so (built by oracle/build_ref.sh from the unmodified
reference sources + a 2-line const fix) and exposes the reference's Model /
AdamW / moe_dispatch / primitive semantics to Python tests and to bench.py's
CPU-baseline leg. Never imported by the product package.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libp2r_ref.so")


class RefConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "d_model", "d_ff", "n_layers_graph", "n_layers_params", "n_heads", "vocab_size",
        "seq_len", "n_experts", "n_prototypes", "n_shards")] + [("capacity_factor", ctypes.c_float)]


@dataclass
class Config:
    """Mirror of p2r::ModelConfig + MoEConfig (model.hpp:13-41), same defaults."""
    d_model: int = 128
    d_ff: int = 512
    n_layers_graph: int = 8
    n_layers_params: int = 8
    n_heads: int = 4
    vocab_size: int = 260
    seq_len: int = 64
    n_experts: int = 0
    n_prototypes: int = 1
    n_shards: int = 1
    capacity_factor: float = 1.25

    def c(self) -> RefConfig:
        return RefConfig(self.d_model, self.d_ff, self.n_layers_graph, self.n_layers_params,
                         self.n_heads, self.vocab_size, self.seq_len, self.n_experts,
                         self.n_prototypes, self.n_shards, self.capacity_factor)

    def shared(self) -> bool:
        return self.n_layers_params == 1 and self.n_layers_graph > 1


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        L = ctypes.CDLL(LIB_PATH)
        vp, ip, fp, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_int64
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_model_create.restype = vp
        L.ref_model_create.argtypes = [ctypes.POINTER(RefConfig), ctypes.c_uint64]
        L.ref_model_destroy.argtypes = [vp]
        L.ref_model_num_params.argtypes = [vp]
        L.ref_model_param_info.argtypes = [vp, ip, ctypes.c_char_p, ctypes.POINTER(ip),
                                           ctypes.POINTER(ip), ctypes.POINTER(i64)]
        for n in ("ref_model_get_param", "ref_model_set_param", "ref_model_get_grad"):
            getattr(L, n).argtypes = [vp, ip, vp]
        L.ref_forward_logits.argtypes = [vp, vp, ip, ip, ip, vp]
        L.ref_train_step.argtypes = [vp, vp, vp, vp, ip, ip, ctypes.c_double, ip, ip, ip, vp]
        L.ref_flush.argtypes = [vp]
        L.ref_scratch_grad_bytes.argtypes = [vp]
        L.ref_scratch_grad_bytes.restype = i64
        L.ref_model_delinked.argtypes = [vp]
        L.ref_model_delinked.restype = vp
        L.ref_adamw_attach.argtypes = [vp, fp, fp, fp, fp]
        L.ref_adamw_step.argtypes = [vp, fp]
        L.ref_adamw_step_count.argtypes = [vp]
        L.ref_adamw_step_count.restype = i64
        L.ref_adamw_set_step_count.argtypes = [vp, i64]
        L.ref_adamw_get_moment.argtypes = [vp, ctypes.c_char_p, ip, vp]
        L.ref_adamw_set_moment.argtypes = [vp, ctypes.c_char_p, ip, vp]
        L.ref_lr_at.argtypes = [fp, ctypes.c_double, i64, i64]
        L.ref_lr_at.restype = fp
        L.ref_count_params.argtypes = [ctypes.POINTER(RefConfig), vp]
        L.ref_moe_dispatch.argtypes = [vp, ip, ip, ip, fp, vp, vp, vp, vp, vp, vp,
                                       ctypes.POINTER(ip), ctypes.POINTER(ip)]
        L.ref_layernorm.argtypes = [vp, vp, vp, ip, ip, vp, vp, vp, vp, vp]
        L.ref_attention.argtypes = [vp, vp, vp, ip, ip, ip, ip, ip, vp, vp, vp, vp, vp]
        L.ref_cross_entropy.argtypes = [vp, vp, vp, ip, ip, ctypes.c_double, vp, vp]
        L.ref_gelu.argtypes = [vp, ip, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _chk(rc):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        exc = {1: ValueError, 2: IndexError, 3: RuntimeError}.get(rc, RuntimeError)
        raise exc(msg)


def count_params(cfg: Config):
    out = np.zeros(3, np.int64)
    _chk(lib().ref_count_params(ctypes.byref(cfg.c()), _p(out)))
    return tuple(int(x) for x in out)


class RefModel:
    """p2r::Model (model.hpp:91-157) + optional p2r::AdamW (optim.hpp:29-54)."""

    def __init__(self, cfg: Config, seed: int = 1234, handle=None):
        self.cfg = cfg
        self.h = handle if handle is not None else lib().ref_model_create(ctypes.byref(cfg.c()), seed)
        if not self.h:
            raise ValueError(lib().ref_last_error().decode())
        self.names, self.shapes = [], []
        name = ctypes.create_string_buffer(128)
        nd, shp, ne = ctypes.c_int(), (ctypes.c_int * 4)(), ctypes.c_int64()
        for i in range(lib().ref_model_num_params(self.h)):
            lib().ref_model_param_info(self.h, i, name, ctypes.byref(nd), shp, ctypes.byref(ne))
            self.names.append(name.value.decode())
            self.shapes.append(tuple(shp[j] for j in range(nd.value)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_model_destroy(self.h)
            self.h = None

    def params(self) -> dict:
        out = {}
        for i, (n, s) in enumerate(zip(self.names, self.shapes)):
            a = np.empty(s, np.float32)
            lib().ref_model_get_param(self.h, i, _p(a))
            out[n] = a
        return out

    def set_params(self, params: dict):
        for i, n in enumerate(self.names):
            a = np.ascontiguousarray(params[n], dtype=np.float32)
            lib().ref_model_set_param(self.h, i, _p(a))

    def grads(self) -> dict:
        out = {}
        for i, (n, s) in enumerate(zip(self.names, self.shapes)):
            a = np.empty(s, np.float32)
            lib().ref_model_get_grad(self.h, i, _p(a))
            out[n] = a
        return out

    def forward(self, tokens: np.ndarray, batch: int, causal: bool = True) -> np.ndarray:
        tok = np.ascontiguousarray(tokens, np.int32)
        out = np.empty((tok.size, self.cfg.vocab_size), np.float32)
        _chk(lib().ref_forward_logits(self.h, _p(tok), batch, tok.size // batch, int(causal), _p(out)))
        return out

    def train_step(self, tokens, targets, mask, batch, denom, causal=True, zero=True,
                   segmented=False) -> float:
        tok = np.ascontiguousarray(tokens, np.int32)
        tgt = np.ascontiguousarray(targets, np.int32)
        msk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        loss = np.zeros(1, np.float32)
        _chk(lib().ref_train_step(self.h, _p(tok), _p(tgt), _p(msk), batch, tok.size // batch,
                                  float(denom), int(causal), int(zero), int(segmented), _p(loss)))
        return float(loss[0])

    def scratch_grad_bytes(self) -> int:
        return int(lib().ref_scratch_grad_bytes(self.h))

    def delinked(self) -> "RefModel":
        h = lib().ref_model_delinked(self.h)
        if not h:
            raise RuntimeError(lib().ref_last_error().decode())
        cfg = Config(**{**self.cfg.__dict__, "n_layers_params": self.cfg.n_layers_graph})
        return RefModel(cfg, handle=h)

    # optimizer
    def attach_adamw(self, b1=0.9, b2=0.999, eps=1e-8, wd=0.01):
        lib().ref_adamw_attach(self.h, b1, b2, eps, wd)

    def adamw_step(self, lr: float):
        _chk(lib().ref_adamw_step(self.h, lr))

    def step_count(self) -> int:
        return int(lib().ref_adamw_step_count(self.h))

    def moments(self) -> dict:
        out = {}
        for n, s in zip(self.names, self.shapes):
            m, v = np.empty(s, np.float32), np.empty(s, np.float32)
            _chk(lib().ref_adamw_get_moment(self.h, n.encode(), 0, _p(m)))
            _chk(lib().ref_adamw_get_moment(self.h, n.encode(), 1, _p(v)))
            out[n] = (m, v)
        return out


def lr_at(peak, warmup_ratio, total, step) -> float:
    return float(lib().ref_lr_at(peak, warmup_ratio, total, step))


@dataclass
class Routing:
    """p2r::Routing (model.hpp:77-87), expert_rows/slots flattened CSR-style."""
    selected: np.ndarray
    survived: np.ndarray
    raw_load: np.ndarray
    offsets: np.ndarray
    rows: np.ndarray
    slots: np.ndarray
    capacity: int
    dropped: int
    expert_rows: list = field(default_factory=list)
    expert_slots: list = field(default_factory=list)


def moe_dispatch(logits: np.ndarray, n_experts: int, n_prototypes: int = 1,
                 capacity_factor: float = 1.25) -> Routing:
    lg = np.ascontiguousarray(logits, np.float32)
    T = lg.shape[0]
    k = n_prototypes
    sel = np.empty(T * k, np.int32)
    sur = np.empty(T * k, np.uint8)
    raw = np.empty(n_experts, np.int32)
    off = np.empty(n_experts + 1, np.int32)
    rows = np.empty(max(T * k, 1), np.int32)
    slots = np.empty(max(T * k, 1), np.int32)
    cap, drop = ctypes.c_int(), ctypes.c_int()
    _chk(lib().ref_moe_dispatch(_p(lg), T, n_experts, k, capacity_factor, _p(sel), _p(sur), _p(raw),
                                _p(off), _p(rows), _p(slots), ctypes.byref(cap), ctypes.byref(drop)))
    n = int(off[-1])
    r = Routing(sel, sur, raw, off, rows[:n].copy(), slots[:n].copy(), cap.value, drop.value)
    r.expert_rows = [r.rows[off[e]:off[e + 1]] for e in range(n_experts)]
    r.expert_slots = [r.slots[off[e]:off[e + 1]] for e in range(n_experts)]
    return r


def layernorm(x, gain, bias, gy):
    x = np.ascontiguousarray(x, np.float32)
    rows, d = x.shape
    y, gx = np.empty_like(x), np.empty_like(x)
    gg, gb = np.empty(d, np.float32), np.empty(d, np.float32)
    _chk(lib().ref_layernorm(_p(x), _p(np.ascontiguousarray(gain, np.float32)),
                             _p(np.ascontiguousarray(bias, np.float32)), rows, d,
                             _p(np.ascontiguousarray(gy, np.float32)), _p(y), _p(gx), _p(gg), _p(gb)))
    return y, gx, gg, gb


def attention(q, k, v, go, causal=True):
    q, k, v, go = (np.ascontiguousarray(t, np.float32) for t in (q, k, v, go))
    B, H, S, hd = q.shape
    o, gq, gk, gv = (np.empty_like(q) for _ in range(4))
    _chk(lib().ref_attention(_p(q), _p(k), _p(v), B, H, S, hd, int(causal), _p(go), _p(o), _p(gq),
                             _p(gk), _p(gv)))
    return o, gq, gk, gv


def cross_entropy(logits, targets, mask, denom):
    lg = np.ascontiguousarray(logits, np.float32)
    rows, V = lg.shape
    loss = np.zeros(1, np.float32)
    g = np.empty_like(lg)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
    _chk(lib().ref_cross_entropy(_p(lg), _p(np.ascontiguousarray(targets, np.int32)), _p(m), rows, V,
                                 float(denom), _p(loss), _p(g)))
    return float(loss[0]), g


def gelu(x, gy):
    x = np.ascontiguousarray(x, np.float32).ravel()
    y, gx = np.empty_like(x), np.empty_like(x)
    _chk(lib().ref_gelu(_p(x), x.size, _p(np.ascontiguousarray(gy, np.float32).ravel()), _p(y), _p(gx)))
    return y, gx
