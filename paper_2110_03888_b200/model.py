"""Python mirror of the reference's Model / AdamW / moe_dispatch surface
(/root/reference/proj/core/include/p2r/model.hpp, optim.hpp) over the C-ABI in
include/p2r_engine.h. Method names match oracle/ref.RefModel so parity tests
read the same against either side. All compute runs in libp2r.so (sm_100a);
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib

vp, ip, fp, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_int64



class PendingLoss:
    """Loss of an enqueued host step (Model.train_step(wait=False)); value() waits for
    that step. Only the two most recent host steps of a model can be waited on."""

    def __init__(self, model, ticket: int):
        self._m, self._t, self._v = model, ticket, None

    def value(self) -> float:
        if self._v is None:
            loss = ctypes.c_float()
            check(lib().p2r_model_loss_wait(self._m.h, ctypes.c_uint64(self._t), ctypes.byref(loss)))
            self._v = float(loss.value)
        return self._v

class ModelConfigC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "d_model", "d_ff", "n_layers_graph", "n_layers_params", "n_heads", "vocab_size",
        "seq_len", "n_experts", "n_prototypes", "n_shards")] + [("capacity_factor", ctypes.c_float)]


class StageStateC(ctypes.Structure):
    """p2r_stage_state (SPEC.md:250-254 StageState)."""
    _fields_ = [("stage", ctypes.c_int), ("global_step", ctypes.c_int64), ("samples_consumed", ctypes.c_int64),
                ("wall_time_s", ctypes.c_double), ("rng_state", ctypes.c_uint64), ("last_eval_step", ctypes.c_int64)]


def _state_dict(s: StageStateC) -> dict:
    return {"stage": "REAL" if s.stage else "PSEUDO", "global_step": s.global_step,
            "samples_consumed": s.samples_consumed, "wall_time_s": s.wall_time_s, "rng_state": s.rng_state,
            "last_eval_step": s.last_eval_step}


_lib._EXTRA_SIGNATURES.update({
    "p2r_count_params": [ctypes.POINTER(ModelConfigC), vp],
    "p2r_model_create": [ctypes.POINTER(ModelConfigC), ctypes.c_uint64, ctypes.POINTER(vp)],
    "p2r_model_destroy": [vp],
    "p2r_model_param_info": [vp, ip, ctypes.c_char_p, ctypes.POINTER(ip), vp, ctypes.POINTER(i64)],
    "p2r_model_get_param": [vp, ip, vp],
    "p2r_model_set_param": [vp, ip, vp],
    "p2r_model_get_grad": [vp, ip, vp],
    "p2r_model_forward": [vp, vp, ip, ip, ip, vp],
    "p2r_model_train_step": [vp, vp, vp, vp, ip, ip, ctypes.c_double, ip, ip, vp],
    "p2r_model_train_step_async": [vp, vp, vp, vp, ip, ip, ctypes.c_double, ip, ip, vp],
    "p2r_model_loss_wait": [vp, ctypes.c_uint64, vp],
    "p2r_model_train_step_device": [vp, vp, vp, vp, ip, ip, ctypes.c_double, ip, ip, vp],
    "p2r_model_train_step_device_graph": [vp, vp, vp, vp, ip, ip, ctypes.c_double, ip, ip, vp],
    "p2r_model_adamw_attach": [vp, fp, fp, fp, fp],
    "p2r_model_adamw_step": [vp, fp],
    "p2r_model_adamw_set_step_count": [vp, i64],
    "p2r_model_get_moment": [vp, ip, ip, vp],
    "p2r_model_delinked": [vp, ctypes.POINTER(vp)],
    "p2r_model_set_moment": [vp, ip, ip, vp],
    "p2r_model_save_checkpoint": [vp, ctypes.c_char_p, ctypes.POINTER(StageStateC)],
    "p2r_model_load_checkpoint": [vp, ctypes.c_char_p, ctypes.POINTER(StageStateC)],
    "p2r_model_from_checkpoint": [ctypes.c_char_p, ctypes.POINTER(vp), ctypes.POINTER(StageStateC)],
    "p2r_delink_checkpoint": [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(StageStateC)],
    "p2r_model_expert_shard": [vp, ip, ctypes.POINTER(ip)],
    "p2r_model_redistribute_experts": [vp, ip],
    "p2r_redistribute_checkpoints": [ctypes.POINTER(ctypes.c_char_p), ip, ctypes.POINTER(ctypes.c_char_p), ip],
    "p2r_model_routing": [vp, ip, vp, vp, vp, ctypes.POINTER(ip), ctypes.POINTER(ip)],
    "p2r_model_gate_logits": [vp, ip, vp],
    "p2r_moe_dispatch_host": [vp, ip, ip, ip, fp, vp, vp, vp, vp, vp, vp,
                              ctypes.POINTER(ip), ctypes.POINTER(ip)],
    "p2r_comm_unique_id": [ctypes.c_char_p],
    "p2r_model_create_ep": [ctypes.POINTER(ModelConfigC), ctypes.c_uint64, ip, ip, ctypes.POINTER(vp)],
    "p2r_model_comm_init": [vp, ctypes.c_char_p],
    "p2r_loopback_create": [ip, ctypes.POINTER(vp)],
    "p2r_loopback_destroy": [vp],
    "p2r_model_comm_init_loopback": [vp, vp],
    "p2r_model_allreduce_grads": [vp],
    "p2r_model_create_offload": [ctypes.POINTER(ModelConfigC), ctypes.c_uint64, vp, ip, ctypes.POINTER(vp)],
    "p2r_model_set_offload_lr": [vp, fp],
    "p2r_model_create_offload_ep": [ctypes.POINTER(ModelConfigC), ctypes.c_uint64, vp, ip, ip, ip,
                                    ctypes.POINTER(vp)],
    "p2r_model_set_grad_accumulation": [vp, ip],
    "p2r_model_set_activation_checkpointing": [vp, ip],
    "p2r_model_offload_stats": [vp, vp],
    "p2r_model_offload_stats_reset": [vp],
    "p2r_model_set_offload_skip_copies": [vp, ip],
    "p2r_plan_offload": [vp, ip, i64, ctypes.c_double, ctypes.c_double, ctypes.c_double, vp],
    "p2r_model_set_profiling": [vp, ip],
    "p2r_model_profile": [vp, ip, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double),
                          ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
    "p2r_model_profile_reset": [vp],
    "p2r_model_buffer": [vp, ip, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t)],
})


def _declare_extra():
    L = lib()
    L.p2r_model_num_params.argtypes = [vp]
    L.p2r_model_num_params.restype = ctypes.c_int
    L.p2r_model_adamw_step_count.argtypes = [vp]
    L.p2r_model_adamw_step_count.restype = i64
    for n in ("p2r_model_state_bytes", "p2r_model_grad_bytes", "p2r_model_scratch_grad_bytes"):
        getattr(L, n).argtypes = [vp]
        getattr(L, n).restype = i64
    L.p2r_model_stream.argtypes = [vp]
    L.p2r_model_stream.restype = vp
    L.p2r_lr_at.argtypes = [fp, ctypes.c_double, i64, i64]
    L.p2r_lr_at.restype = fp
    L.p2r_moe_capacity.argtypes = [fp, ip, ip, ip]
    L.p2r_moe_capacity.restype = ctypes.c_int
    for n in ("p2r_model_layer_granule_bytes", "p2r_model_device_param_bytes"):
        getattr(L, n).argtypes = [vp]
        getattr(L, n).restype = i64
    L.p2r_predict_step_time.argtypes = [vp, vp, ip, ctypes.c_double, ctypes.c_double, ctypes.c_double]
    L.p2r_predict_step_time.restype = ctypes.c_double
    L.p2r_predict_step_time_overlap.argtypes = [vp, vp, vp, ip] + [ctypes.c_double] * 4
    L.p2r_predict_step_time_overlap.restype = ctypes.c_double
    L.p2r_predict_step_time_overlap_form.argtypes = [vp, vp, vp, ip] + [ctypes.c_double] * 4 + [ip]
    L.p2r_predict_step_time_overlap_form.restype = ctypes.c_double
    L.p2r_predict_step_time_overlap_window.argtypes = [vp, vp, vp, ip] + [ctypes.c_double] * 4 + [ip, ip, ip]
    L.p2r_predict_step_time_overlap_window.restype = ctypes.c_double
    L.p2r_plan_offload_overlap.argtypes = [vp, ip, i64] + [ctypes.c_double] * 4 + [ip, vp]
    L.p2r_plan_offload_overlap.restype = ctypes.c_int
    return L


def comm_unique_id() -> bytes:
    """ncclGetUniqueId: 128 bytes to broadcast to every rank before Model.comm_init."""
    _declare_extra()
    buf = ctypes.create_string_buffer(128)
    check(lib().p2r_comm_unique_id(buf))
    return buf.raw


def plan_offload(layer_bytes, budget, bandwidth, compute_s, latency_s=0.0):
    """plan_offload -> list of 0/1 (1 = SLOW / offloaded)."""
    _declare_extra()
    b = np.ascontiguousarray(layer_bytes, np.int64)
    out = np.zeros(b.size, np.int32)
    check(lib().p2r_plan_offload(_p(b), b.size, int(budget), float(bandwidth), float(compute_s),
                                 float(latency_s), _p(out)))
    return [int(x) for x in out]


def predict_step_time(layer_bytes, slow, bandwidth, compute_s, latency_s=0.0) -> float:
    L = _declare_extra()
    b = np.ascontiguousarray(layer_bytes, np.int64)
    s = np.ascontiguousarray(slow, np.int32)
    return float(L.p2r_predict_step_time(_p(b), _p(s), b.size, float(bandwidth), float(compute_s),
                                         float(latency_s)))


def _p(a):
    return None if a is None else a.ctypes.data_as(vp)


@dataclass
class Config:
    """ModelConfig + MoEConfig (model.hpp:13-41), same fields and defaults."""
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

    def c(self) -> ModelConfigC:
        return ModelConfigC(self.d_model, self.d_ff, self.n_layers_graph, self.n_layers_params,
                            self.n_heads, self.vocab_size, self.seq_len, self.n_experts,
                            self.n_prototypes, self.n_shards, self.capacity_factor)

    def shared(self) -> bool:
        return self.n_layers_params == 1 and self.n_layers_graph > 1

    def as_unshared(self) -> "Config":
        return Config(**{**self.__dict__, "n_layers_params": self.n_layers_graph})


def count_params(cfg: Config):
    _declare_extra()
    out = np.zeros(3, np.int64)
    check(lib().p2r_count_params(ctypes.byref(cfg.c()), _p(out)))
    return tuple(int(x) for x in out)


def lr_at(peak, warmup_ratio, total, step) -> float:
    return float(_declare_extra().p2r_lr_at(peak, warmup_ratio, total, step))


class Model:
    """p2r::Model + AdamW on one B200 (one CUDA stream per model)."""

    def __init__(self, cfg: Config, seed: int = 1234, handle=None, offload=None, ring_slots: int = 3,
                 ep=None):
        """offload: per-owned-layer 0/1 placement (1 = SLOW, kept in pinned host DRAM).
        ep: (world, rank) expert-parallel shard (call comm_init before stepping)."""
        L = _declare_extra()
        self.cfg = cfg
        if handle is None:
            h = vp()
            if ep is not None and offload is not None:
                sl = np.ascontiguousarray(offload, np.int32)
                check(L.p2r_model_create_offload_ep(ctypes.byref(cfg.c()), seed, _p(sl), ring_slots, int(ep[0]),
                                                    int(ep[1]), ctypes.byref(h)))
            elif ep is not None:
                check(L.p2r_model_create_ep(ctypes.byref(cfg.c()), seed, int(ep[0]), int(ep[1]),
                                            ctypes.byref(h)))
            elif offload is None:
                check(L.p2r_model_create(ctypes.byref(cfg.c()), seed, ctypes.byref(h)))
            else:
                sl = np.ascontiguousarray(offload, np.int32)
                check(L.p2r_model_create_offload(ctypes.byref(cfg.c()), seed, _p(sl), ring_slots,
                                                 ctypes.byref(h)))
            handle = h.value
        self.h = handle
        self.names, self.shapes = [], []
        name = ctypes.create_string_buffer(128)
        nd, shp, ne = ctypes.c_int(), (ctypes.c_int * 4)(), ctypes.c_int64()
        for i in range(L.p2r_model_num_params(self.h)):
            check(L.p2r_model_param_info(self.h, i, name, ctypes.byref(nd), shp, ctypes.byref(ne)))
            self.names.append(name.value.decode())
            self.shapes.append(tuple(shp[j] for j in range(nd.value)))

    def close(self):
        if getattr(self, "h", None):
            lib().p2r_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- parameters (for_each_param order)
    def _get(self, fn, i, shape):
        a = np.empty(shape, np.float32)
        check(fn(self.h, i, _p(a)))
        return a

    def params(self) -> dict:
        return {n: self._get(lib().p2r_model_get_param, i, s)
                for i, (n, s) in enumerate(zip(self.names, self.shapes))}

    def set_params(self, params: dict):
        for i, n in enumerate(self.names):
            a = np.ascontiguousarray(params[n], dtype=np.float32)
            check(lib().p2r_model_set_param(self.h, i, _p(a)))

    def grads(self) -> dict:
        return {n: self._get(lib().p2r_model_get_grad, i, s)
                for i, (n, s) in enumerate(zip(self.names, self.shapes))}

    def moments(self) -> dict:
        out = {}
        for i, (n, s) in enumerate(zip(self.names, self.shapes)):
            m = np.empty(s, np.float32)
            v = np.empty(s, np.float32)
            check(lib().p2r_model_get_moment(self.h, i, 0, _p(m)))
            check(lib().p2r_model_get_moment(self.h, i, 1, _p(v)))
            out[n] = (m, v)
        return out

    def set_moments(self, moments: dict):
        for i, n in enumerate(self.names):
            m, v = (np.ascontiguousarray(x, dtype=np.float32) for x in moments[n])
            check(lib().p2r_model_set_moment(self.h, i, 0, _p(m)))
            check(lib().p2r_model_set_moment(self.h, i, 1, _p(v)))

    # ---- checkpoint container (csrc/engine/checkpoint.cpp)
    def save_checkpoint(self, path: str, stage: str = None, global_step: int = 0, samples_consumed: int = 0,
                        wall_time_s: float = 0.0, rng_state: int = 0, last_eval_step: int = -1):
        """Parameters, AdamW moments + step count and the StageState. stage defaults to
        PSEUDO for a shared-parameter model and REAL otherwise."""
        if stage is None:
            stage = "PSEUDO" if self.cfg.shared() else "REAL"
        if stage not in ("PSEUDO", "REAL"):
            raise ValueError("stage must be PSEUDO or REAL")
        st = StageStateC(1 if stage == "REAL" else 0, global_step, samples_consumed, wall_time_s, rng_state,
                         last_eval_step)
        check(lib().p2r_model_save_checkpoint(self.h, path.encode(), ctypes.byref(st)))

    def load_checkpoint(self, path: str) -> dict:
        """Load into this model (same config); returns the StageState as a dict."""
        st = StageStateC()
        check(lib().p2r_model_load_checkpoint(self.h, path.encode(), ctypes.byref(st)))
        return _state_dict(st)

    # ---- expert sharding bookkeeping (model.cpp:334-356)
    def expert_shard(self, expert: int) -> int:
        out = ctypes.c_int()
        check(lib().p2r_model_expert_shard(self.h, expert, ctypes.byref(out)))
        return out.value

    def shard_layout(self):
        return [[e for e in range(self.cfg.n_experts) if self.expert_shard(e) == s]
                for s in range(self.cfg.n_shards)]

    def redistribute_experts(self, new_n_shards: int):
        check(lib().p2r_model_redistribute_experts(self.h, new_n_shards))
        self.cfg = Config(**{**self.cfg.__dict__, "n_shards": new_n_shards})

    # ---- compute
    def forward(self, tokens, batch: int, causal: bool = True) -> np.ndarray:
        tok = np.ascontiguousarray(tokens, np.int32)
        out = np.empty((tok.size, self.cfg.vocab_size), np.float32)
        check(lib().p2r_model_forward(self.h, _p(tok), batch, tok.size // batch, int(causal), _p(out)))
        return out

    def train_step(self, tokens, targets, mask, batch, denom, causal=True, zero=True,
                   segmented=False, wait=True):
        """One micro-step on host arrays; returns the loss. wait=False returns a
        PendingLoss at once (the step and its loss read-back are enqueued), so a
        training loop can enqueue the optimizer / next step before reading it."""
        del segmented  # one fused backward; equivalent to the reference's segmented variant
        tok = np.ascontiguousarray(tokens, np.int32)
        tgt = np.ascontiguousarray(targets, np.int32)
        msk = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        if not wait:
            ticket = ctypes.c_uint64()
            check(lib().p2r_model_train_step_async(self.h, _p(tok), _p(tgt), _p(msk), batch, tok.size // batch,
                                                   float(denom), int(causal), int(zero), ctypes.byref(ticket)))
            return PendingLoss(self, ticket.value)
        loss = ctypes.c_float()
        check(lib().p2r_model_train_step(self.h, _p(tok), _p(tgt), _p(msk), batch, tok.size // batch,
                                         float(denom), int(causal), int(zero), ctypes.byref(loss)))
        return float(loss.value)

    def train_step_device(self, d_tokens: int, d_targets: int, d_mask, batch: int, seq: int,
                          denom: float, causal=True, zero=True, loss_dev=None, graph=False):
        """Inputs resident on the device. graph=True replays the step as one CUDA
        graph (captured on first use; resident, MoE-free models)."""
        fn = lib().p2r_model_train_step_device_graph if graph else lib().p2r_model_train_step_device
        check(fn(self.h, d_tokens, d_targets, d_mask, batch, seq, float(denom), int(causal), int(zero), loss_dev))

    def stream(self) -> int:
        return int(lib().p2r_model_stream(self.h) or 0)

    # ---- expert / data parallelism (NCCL)
    def comm_init(self, unique_id: bytes):
        check(lib().p2r_model_comm_init(self.h, ctypes.c_char_p(unique_id)))

    def comm_init_loopback(self, group: "LoopbackGroup"):
        """Join a loopback group (W shards of this process on one device; drive each
        shard's steps from its own thread -- the exchange is collective)."""
        check(lib().p2r_model_comm_init_loopback(self.h, group.h))
        self._group = group  # keep the group alive as long as its shards

    def allreduce_grads(self):
        check(lib().p2r_model_allreduce_grads(self.h))

    # ---- granular offload
    def set_offload_lr(self, lr: float):
        check(lib().p2r_model_set_offload_lr(self.h, lr))

    def set_grad_accumulation(self, micro_steps: int):
        check(lib().p2r_model_set_grad_accumulation(self.h, micro_steps))

    def set_activation_checkpointing(self, policy: int):
        """0 off, 1 SLOW layers (default for offloaded models), 2 every layer."""
        check(lib().p2r_model_set_activation_checkpointing(self.h, policy))

    def offload_stats(self) -> dict:
        o = np.zeros(8, np.float64)
        check(lib().p2r_model_offload_stats(self.h, _p(o)))
        keys = ("Fn_load", "Bn_load", "opt_load", "writeback", "grad_offload", "h2d_ms", "d2h_ms", "grad_load")
        return dict(zip(keys, (float(x) for x in o)))

    def offload_stats_reset(self):
        check(lib().p2r_model_offload_stats_reset(self.h))

    def set_offload_skip_copies(self, skip: bool):
        check(lib().p2r_model_set_offload_skip_copies(self.h, int(skip)))

    def layer_granule_bytes(self) -> int:
        return int(lib().p2r_model_layer_granule_bytes(self.h))

    def device_param_bytes(self) -> int:
        return int(lib().p2r_model_device_param_bytes(self.h))

    PROF_CLASSES = ("gemm", "attn_fwd", "attn_bwd", "layernorm", "cross_entropy", "embed", "adamw",
                    "moe", "bias_grad", "delink")

    def set_profiling(self, on: bool):
        check(lib().p2r_model_set_profiling(self.h, int(on)))

    def profile(self) -> dict:
        """{class: (launches, device ms, algorithmic flops, algorithmic bytes)} since last reset."""
        out = {}
        n, ms, fl, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        for i, name in enumerate(self.PROF_CLASSES):
            check(lib().p2r_model_profile(self.h, i, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl),
                                          ctypes.byref(by)))
            out[name] = (int(n.value), float(ms.value), float(fl.value), float(by.value))
        return out

    def profile_reset(self):
        check(lib().p2r_model_profile_reset(self.h))

    def buffer(self, which: int):
        """(device pointer, bytes) of the embeddings (0) / owned-layers (1) gradient granules."""
        p, n = vp(), ctypes.c_size_t()
        check(lib().p2r_model_buffer(self.h, which, ctypes.byref(p), ctypes.byref(n)))
        return int(p.value), int(n.value)

    def scratch_grad_bytes(self) -> int:
        return int(lib().p2r_model_scratch_grad_bytes(self.h))

    def grad_bytes(self) -> int:
        return int(lib().p2r_model_grad_bytes(self.h))

    def state_bytes(self) -> int:
        return int(lib().p2r_model_state_bytes(self.h))

    def delinked(self) -> "Model":
        h = vp()
        check(lib().p2r_model_delinked(self.h, ctypes.byref(h)))
        return Model(self.cfg.as_unshared(), handle=h.value)

    # ---- optimizer
    def attach_adamw(self, b1=0.9, b2=0.999, eps=1e-8, wd=0.01):
        check(lib().p2r_model_adamw_attach(self.h, b1, b2, eps, wd))

    def adamw_step(self, lr: float):
        check(lib().p2r_model_adamw_step(self.h, lr))

    def step_count(self) -> int:
        return int(lib().p2r_model_adamw_step_count(self.h))

    def set_step_count(self, t: int):
        check(lib().p2r_model_adamw_set_step_count(self.h, t))

    def layer_routing(self, g: int, n_tokens: int):
        k = self.cfg.n_prototypes
        sel = np.empty(n_tokens * k, np.int32)
        sur = np.empty(n_tokens * k, np.uint8)
        raw = np.empty(self.cfg.n_experts, np.int32)
        cap, drop = ctypes.c_int(), ctypes.c_int()
        check(lib().p2r_model_routing(self.h, g, _p(sel), _p(sur), _p(raw), ctypes.byref(cap),
                                      ctypes.byref(drop)))
        return sel, sur, raw, cap.value, drop.value

    def gate_logits(self, g: int, n_tokens: int) -> np.ndarray:
        """fp32 gate logits [T, E] of graph layer g from the last forward."""
        out = np.empty((n_tokens, self.cfg.n_experts), np.float32)
        check(lib().p2r_model_gate_logits(self.h, g, _p(out)))
        return out


class LoopbackGroup:
    """W expert/data-parallel shards in one process on one device (SURVEY §4's
    loopback comm): the same peer-store exchange and stream flags as a multi-GPU
    node, with the shards' own arenas as peer memory; rank-order all-reduce."""

    def __init__(self, world: int):
        h = vp()
        check(lib().p2r_loopback_create(int(world), ctypes.byref(h)))
        self.h = h.value
        self.world = world

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().p2r_loopback_destroy(self.h)
                self.h = None
        except Exception:  # noqa: BLE001
            pass


@dataclass
class Routing:
    """p2r::Routing (model.hpp:77-87); expert_rows/slots flattened CSR-style."""
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
    """moe_dispatch (model.cpp:294-332) computed by the sm_100a routing kernel."""
    lg = np.ascontiguousarray(logits, np.float32)
    if lg.ndim != 2 or lg.shape[1] != n_experts:
        raise _lib.P2RInvalidArgument("moe_dispatch: logits must be [tokens, n_experts]")
    T, k = lg.shape[0], n_prototypes
    sel = np.empty(max(T * k, 1), np.int32)
    sur = np.empty(max(T * k, 1), np.uint8)
    raw = np.empty(n_experts, np.int32)
    off = np.empty(n_experts + 1, np.int32)
    rows = np.empty(max(T * k, 1), np.int32)
    slots = np.empty(max(T * k, 1), np.int32)
    cap, drop = ctypes.c_int(), ctypes.c_int()
    _declare_extra()
    check(lib().p2r_moe_dispatch_host(_p(lg), T, n_experts, k, capacity_factor, _p(sel), _p(sur),
                                      _p(raw), _p(off), _p(rows), _p(slots), ctypes.byref(cap),
                                      ctypes.byref(drop)))
    n = int(off[-1])
    r = Routing(sel[:T * k], sur[:T * k], raw, off, rows[:n].copy(), slots[:n].copy(), cap.value,
                drop.value)
    r.expert_rows = [r.rows[off[e]:off[e + 1]] for e in range(n_experts)]
    r.expert_slots = [r.slots[off[e]:off[e + 1]] for e in range(n_experts)]
    return r


def load_checkpoint(path: str):
    """Model.from_checkpoint: returns (Model, StageState dict)."""
    from .checkpoint import read_manifest
    _declare_extra()
    c = read_manifest(path)["config"]
    h, st = vp(), StageStateC()
    check(lib().p2r_model_from_checkpoint(path.encode(), ctypes.byref(h), ctypes.byref(st)))
    return Model(Config(**c), handle=h.value), _state_dict(st)


def delink_checkpoint(in_path: str, out_path: str) -> dict:
    """[OP] delink(pseudo_checkpoint) -> Real checkpoint."""
    _declare_extra()
    st = StageStateC()
    check(lib().p2r_delink_checkpoint(in_path.encode(), out_path.encode(), ctypes.byref(st)))
    return _state_dict(st)


def redistribute_checkpoints(in_paths, out_paths):
    """Re-shard expert-parallel shard checkpoints across GPU counts (len(in_paths) ->
    len(out_paths) shards; weights + AdamW moments; SPEC redistribute_experts)."""
    _declare_extra()
    ins = (ctypes.c_char_p * len(in_paths))(*[p.encode() for p in in_paths])
    outs = (ctypes.c_char_p * len(out_paths))(*[p.encode() for p in out_paths])
    check(lib().p2r_redistribute_checkpoints(ins, len(in_paths), outs, len(out_paths)))


def predict_step_time_overlap(layer_params, slow, h2d_bw, d2h_bw, fwd_s, bwd_s, vector_params=None,
                              fn_master=False, micro_steps=1, recompute=False) -> float:
    """B200 overlap model of the offload engine; see p2r_engine.h.
    fn_master: the engine's default forward load (fp32 master); False = the bf16-shadow form.
    micro_steps / recompute: accumulation window and SLOW-layer checkpoint recomputation."""
    L = _declare_extra()
    p = np.ascontiguousarray(layer_params, np.int64)
    sl = np.ascontiguousarray(slow, np.int32)
    v = None if vector_params is None else np.ascontiguousarray(vector_params, np.int64)
    return float(L.p2r_predict_step_time_overlap_window(_p(p), _p(v), _p(sl), len(p), h2d_bw, d2h_bw, fwd_s, bwd_s,
                                                        int(bool(fn_master)), int(micro_steps), int(bool(recompute))))


def plan_offload_overlap(layer_params, budget_bytes, h2d_bw, d2h_bw, fwd_s, bwd_s, ring_slots=3):
    """Budget covers the resident granules AND the ring_slots HBM staging slots."""
    L = _declare_extra()
    p = np.ascontiguousarray(layer_params, np.int64)
    out = np.zeros(len(p), np.int32)
    check(L.p2r_plan_offload_overlap(_p(p), len(p), int(budget_bytes), h2d_bw, d2h_bw, fwd_s, bwd_s,
                                     int(ring_slots), _p(out)))
    return out.tolist()
