"""B200-native (sm_100a) training-step hot path of arXiv 2110.03888 (Pseudo-to-Real).

The product is libp2r.so: hand-written tcgen05/TMA GEMMs, fused attention,
LayerNorm / CE / AdamW / delink / MoE routing kernels and a C++ host engine
that keeps the reference's Model / AdamW / moe_dispatch API. This package is
a thin ctypes mirror of that API (see model.py); it never computes on the CPU.
"""
from ._lib import (P2RError, P2RInvalidArgument, P2RLogicError, P2ROutOfRange, launch_count,
                   lib)
from .model import (Config, LoopbackGroup, Model, PendingLoss, Routing, comm_unique_id, count_params,
                    delink_checkpoint, load_checkpoint, lr_at, moe_dispatch, plan_offload, plan_offload_overlap, predict_step_time,
                    predict_step_time_overlap, redistribute_checkpoints)

__all__ = ["Config", "LoopbackGroup", "Model", "PendingLoss", "Routing", "count_params", "lr_at", "moe_dispatch", "plan_offload",
           "predict_step_time", "load_checkpoint", "delink_checkpoint", "redistribute_checkpoints", "plan_offload_overlap",
           "predict_step_time_overlap", "lib",
           "launch_count", "P2RError", "P2RInvalidArgument", "P2ROutOfRange", "P2RLogicError"]
