#!/usr/bin/env python
"""Training-step benchmark of the Pseudo-to-Real hot path on B200.

Default workload (BASELINE.json configs[1], "C2"): pseudo-giant dense GPT block
shared across 24 layers, d=1024, 16 heads, d_ff=4096, seq 1024, batch 8
sequences per GPU, vocab 260, random-init weights (reference init, seed 1234),
synthetic byte tokens. One step = embed -> 24 x block fwd -> tied head -> masked
CE -> full backward (shared-layer grads accumulated in place) -> [NCCL
allreduce of the shared + embedding grads when N > 1] -> AdamW.

  python bench.py [--gpus N --steps K --warmup W]          # this framework
  python bench.py --impl reference [...]                    # reference CPU arm
  python bench.py --workload c3|c4|c5 [...]                 # the other configs

--gpus N > 1 without torchrun's WORLD_SIZE re-launches itself under
torch.distributed.run with N ranks. Other workloads (BASELINE.json configs):
  c3  Pseudo MoE (24 shared layers, d=1024, 8 experts top-1) delinked into the
      Real model, then the Real step; experts sharded over the N GPUs
  c4  M6-style MoE per-rank slice: d=2048, 8 experts per GPU (64 at N=8), top-1,
      --layers (48), expert parallel over the N GPUs
  c5  granular-offload per-rank slice (d=2048, 8 local experts, --layers 8,
      half the layers SLOW, 2-micro-step accumulation): resident / offload /
      offload-without-copies steps, PCIe GB/s per direction and hidden fraction

Prints ONE JSON line on rank 0. `value` = tokens/s over all ranks with inputs
resident in HBM (CUDA events on the model stream around the K timed steps, max
over ranks); `e2e` = the same metric through the public host-buffer API
(tokens/targets/mask copied in from pinned memory, loss read back, every step;
a pipelined loop: step i+1 and its AdamW are enqueued before step i's loss is read).
`roofline` comes from a SEPARATE eager pass of K more steps in which every
kernel is bracketed by CUDA events on the model stream (per-class time and
algorithmic FLOPs/bytes); it explains `value` but is not part of its timed
region. `cpu_baseline` times the compiled reference (oracle/_ref) on the host
cores on a bounded sample. The default C2 line also carries two in-run
sub-records: `moe_ep` (C4 per-rank slice, local vs expert-parallel exchange
path) and `offload` (C5 per-rank slice, hidden fraction of the PCIe traffic).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(d_model=1024, d_ff=4096, n_layers_graph=24, n_layers_params=1, n_heads=16,
          vocab_size=260, seq_len=1024)
WORKLOAD = ("C2 pseudo-giant dense GPT block shared x24 (d=1024, 16 heads, d_ff=4096, "
            "vocab 260, seq 1024), fwd+bwd+AdamW")
METRIC = "train tokens/sec"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="p2r", choices=["p2r", "reference"])
    p.add_argument("--batch", type=int, default=8)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph per step")
    p.add_argument("--cpu-procs", type=int, default=0, help="reference processes (0 = auto)")
    p.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    p.add_argument("--layers", type=int, default=0, help="c3/c4/c5: layer count (0 = the config's)")
    p.add_argument("--no-extras", action="store_true", help="c2: skip the moe_ep / offload sub-records")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def lm_batch(batch, seq, seed):
    """make_lm_batch semantics (data.cpp:174-195) on synthetic byte tokens."""
    rng = np.random.default_rng(seed)
    tok = rng.integers(0, 256, (batch, seq)).astype(np.int32)
    tgt = np.zeros_like(tok)
    tgt[:, :-1] = tok[:, 1:]
    mask = np.ones_like(tok, dtype=np.uint8)
    mask[:, -1] = 0
    return tok.ravel(), tgt.ravel(), mask.ravel()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except (OSError, ValueError):
        return dict(FALLBACK_PEAKS), "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU reference
def _ref_worker(args):
    """One reference micro-step (fwd+bwd+AdamW) of the C2 model on one sequence."""
    seq, nlayers, seed = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ.setdefault("OPENBLAS_CORETYPE", "SkylakeX")
    from oracle import ref
    cfg = ref.Config(**dict(C2, n_layers_graph=nlayers))
    m = _ref_worker.cache.get((seq, nlayers))
    if m is None:
        m = ref.RefModel(cfg, 1234)
        m.attach_adamw()
        _ref_worker.cache[(seq, nlayers)] = m
    tok, tgt, mask = lm_batch(1, seq, seed)
    t0 = time.perf_counter()
    m.train_step(tok, tgt, mask, 1, float(mask.sum()))
    m.adamw_step(1e-5)
    return time.perf_counter() - t0


_ref_worker.cache = {}


def ref_procs(requested):
    if requested > 0:
        return requested
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        import psutil
        avail_gb = psutil.virtual_memory().available / 2**30
    except Exception:  # noqa: BLE001
        avail_gb = 64
    # one reference C2 micro-step on 1024 tokens keeps ~4 GB of fp32 activations
    return max(1, min(ncpu, int(avail_gb * 0.5 / 4.5), 64))


def _ref_loop(conn):
    """Persistent reference worker: builds its model once, then one micro-step per command."""
    while True:
        msg = conn.recv()
        if msg is None:
            conn.close()
            return
        conn.send(_ref_worker(msg))


def run_reference_steps(nproc, steps, warmup):
    """`steps` timed rounds; in each round every process runs exactly one
    1024-token micro-step of the C2 model (round time = slowest process)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    pipes, procs = [], []
    for _ in range(nproc):
        a, b = ctx.Pipe()
        p = ctx.Process(target=_ref_loop, args=(b,), daemon=True)
        p.start()
        pipes.append(a)
        procs.append(p)

    def round_(seed0):
        for i, c in enumerate(pipes):
            c.send((C2["seq_len"], C2["n_layers_graph"], seed0 + i))
        return [c.recv() for c in pipes]

    try:
        for w in range(max(1, warmup)):
            round_(7 + w * nproc)
        t0 = time.perf_counter()
        for s in range(steps):
            round_(1000 + s * nproc)
        dt = time.perf_counter() - t0
    finally:
        for c in pipes:
            c.send(None)
        for p in procs:
            p.join(timeout=30)
    tokens = steps * nproc * C2["seq_len"]
    return tokens / dt, dt / steps


def cpu_baseline_sample(nproc):
    """Bounded sample for the GPU arm's JSON: one round (warm-up excluded) of
    nproc concurrent single-threaded reference micro-steps on 1024 tokens."""
    tps, step_s = run_reference_steps(nproc, 1, 1)
    return {"value": round(tps, 2), "unit": "tokens/s", "cores": nproc, "kind": "reference",
            "sample": (f"{nproc} concurrent single-thread processes, each one fwd+bwd+AdamW micro-step of "
                       f"the full C2 model (24 shared layers) on 1 x 1024 tokens after 1 warm-up round; "
                       f"oracle/_ref/libp2r_ref.so (reference sources, OpenBLAS 0.3.15 SkylakeX, 1 thread); "
                       f"round wall time {step_s:.1f} s")}


def main_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    nproc = ref_procs(args.cpu_procs)
    tps, step_s = run_reference_steps(nproc, args.steps, args.warmup)
    out = {"impl": "reference", "metric": METRIC, "value": round(tps, 2), "unit": "tokens/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(step_s * 1e3, 1), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": WORKLOAD, "global_batch": nproc, "seq_len": C2["seq_len"],
                      "parallelism": f"{nproc} CPU processes"},
           "cpu_baseline": {"value": round(tps, 2), "unit": "tokens/s", "cores": nproc, "kind": "reference",
                            "sample": (f"each step: {nproc} concurrent single-thread reference processes x one "
                                       f"1024-token fwd+bwd+AdamW micro-step of the C2 model")},
           "e2e": {"value": round(tps, 2), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def moe_cfg(p2r, d, dff, heads, layers, params, experts, seq):
    return p2r.Config(d_model=d, d_ff=dff, n_layers_graph=layers, n_layers_params=params, n_heads=heads,
                      vocab_size=260, seq_len=seq, n_experts=experts, n_prototypes=1)


def flops_per_token(d, dff, L, S, V=260, E=0, k_eff=1.0):
    """§8(d): 3 x [L (8d^2 + 4 k_eff d dff + 2 d E + 2 S d) + 2 d V] (fwd + bwd, no recompute)."""
    return 3 * (L * (8 * d * d + 4 * k_eff * d * dff + 2 * d * E + 2 * S * d) + 2 * d * V)


def make_dist(world, local):
    import torch
    if world <= 1:
        return None
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist


def comm_init(model, p2r, dist, rank, world):
    if world > 1:
        # the library's own NCCL communicator (csrc/engine/comm.cpp); torch only ships the id
        uid = [p2r.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        model.comm_init(uid[0])


def build_workload(args, p2r, dist, rank, world):
    """-> (model, batch, seq, workload text, model FLOPs per token, graph ok, parallelism)."""
    B, S = args.batch, 1024
    if args.workload == "c2":
        m = p2r.Model(p2r.Config(**C2), 1234)
        comm_init(m, p2r, dist, rank, world)
        return m, B, S, WORKLOAD, flops_per_token(1024, 4096, 24, S), True, f"dp{world}"
    if args.workload == "c3":
        E = 8
        if E % world:
            raise SystemExit("c3: 8 experts need a GPU count dividing 8")
        L = args.layers or 24
        pseudo = p2r.Model(moe_cfg(p2r, 1024, 4096, 16, L, 1, E, S), 1234, ep=(world, rank))
        real = pseudo.delinked()  # every rank delinks its own shard (no communication)
        pseudo.close()
        comm_init(real, p2r, dist, rank, world)
        text = (f"C3 Pseudo MoE ({L} shared layers, d=1024, 16 heads, d_ff=4096, {E} experts top-1 cf 1.25, "
                f"vocab 260, seq 1024) delinked into {L} Real layers; Real-model fwd+bwd+AdamW, "
                f"experts over {world} GPU(s)")
        return real, B, S, text, flops_per_token(1024, 4096, L, S, E=E), world == 1, f"ep{world}+dp{world}"
    if args.workload == "c4":
        E = 8 * world  # 8 experts per GPU: the C4 per-rank share (64 experts at N = 8)
        L = args.layers or 48
        m = p2r.Model(moe_cfg(p2r, 2048, 4096, 16, L, L, E, S), 1234, ep=(world, rank))
        comm_init(m, p2r, dist, rank, world)
        text = (f"C4 M6-style MoE per-rank slice: {L} Real layers, d=2048, 16 heads, d_ff=4096, 8 experts per GPU "
                f"({E} total) top-1 cf 1.25, vocab 260, seq 1024, fwd+bwd+AdamW")
        return m, B, S, text, flops_per_token(2048, 4096, L, S, E=E), world == 1, f"ep{world}+dp{world}"
    raise SystemExit(f"unknown workload {args.workload}")


def moe_ep_record(p2r, torch, steps=4, warmup=2, layers=4):
    """C4 per-rank slice at `layers` layers: the local expert path vs the expert-parallel
    exchange path at world 1 (peer-store send, owner pack, exact-count GEMMs, return),
    same tokens; ms per step and the bytes the exchange moves."""
    B, S = 8, 1024
    cfg = moe_cfg(p2r, 2048, 4096, 16, layers, layers, 8, S)
    tok, tgt, mask = lm_batch(B, S, 7)
    dt, dg, dm = (torch.from_numpy(x).cuda() for x in (tok, tgt, mask))
    out = {}
    for name in ("local", "ep_w1"):
        if name == "ep_w1":
            os.environ["P2R_FORCE_EP"] = "1"
        try:
            m = p2r.Model(cfg, 1234, ep=(1, 0)) if name == "ep_w1" else p2r.Model(cfg, 1234)
        finally:
            os.environ.pop("P2R_FORCE_EP", None)
        m.attach_adamw()
        ext = torch.cuda.ExternalStream(m.stream())

        def step(i):
            m.train_step_device(dt.data_ptr(), dg.data_ptr(), dm.data_ptr(), B, S, float(mask.sum()))
            m.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, i))

        for i in range(warmup):
            step(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ext):
            e0.record()
        for i in range(steps):
            step(warmup + i)
        with torch.cuda.stream(ext):
            e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        rows = 0
        for g in range(layers):
            sel, sur, raw, cap, drop = m.layer_routing(g, B * S)
            rows += int(sur.sum())
        out[name] = {"ms_per_step": round(ms, 3), "tokens_per_s": round(B * S / (ms / 1e3), 1)}
        if name == "ep_w1":
            # rows cross the link as bf16 in each of the 4 exchanges per layer
            # (fwd dispatch + return, bwd dispatch + return); at W ranks the remote
            # share is (W-1)/W of it
            out["exchange_bytes_per_direction_per_layer"] = int(rows // layers * 2048 * 2)
            out["algorithmic_bytes_T_d_2"] = B * S * 2048 * 2
        m.close()
        del m
        torch.cuda.empty_cache()
    out["ep_over_local"] = round(out["ep_w1"]["ms_per_step"] / out["local"]["ms_per_step"], 4)
    out["workload"] = (f"C4 per-rank slice, {layers} Real layers, d=2048, d_ff=4096, 8 experts top-1, 8x1024 tokens, "
                       f"fwd+bwd+AdamW; CUDA events over {steps} steps after {warmup} warm-up")
    return out


def offload_record(p2r, torch, layers=8, steps=3, warmup=2, ring=6, micro=1, batch=64):
    """C5 per-rank slice: granular offload of half the layers (interleaved, the overlap
    planner's spread), activation checkpointing of SLOW layers, `micro` accumulation
    micro-steps per optimizer step. Resident / offload / offload-without-copies step
    times (CUDA events), copy-engine busy time (events on the H2D / D2H streams) and
    the hidden fraction h = 1 - (T_offload - T_nocopy) / max(T_h2d, T_d2h)."""
    B, S = batch, 1024
    cfg = moe_cfg(p2r, 2048, 4096, 16, layers, layers, 8, S)
    # half the layers SLOW (C5: ~45 of 96 granules do not fit HBM), spread the way the
    # overlap-aware planner spreads them (half a stride in: layer 0 stays resident)
    k = layers // 2
    plan = [0] * layers
    for j in range(k):
        plan[(2 * j + 1) * layers // (2 * k)] = 1
    batches = [tuple(torch.from_numpy(x).cuda() for x in lm_batch(B, S, 50 + j)) for j in range(micro)]
    denom = float(micro * B * (S - 1))

    def run(m, offloaded, n):
        ext = torch.cuda.ExternalStream(m.stream())

        def one(i):
            lr = p2r.lr_at(2e-4, 0.01, 1000, i + 10)
            if offloaded:
                m.set_offload_lr(lr)
            for j, (dt, dg, dm) in enumerate(batches):
                m.train_step_device(dt.data_ptr(), dg.data_ptr(), dm.data_ptr(), B, S, denom, zero=(j == 0))
            m.adamw_step(lr)

        for i in range(warmup):
            one(i)
        torch.cuda.synchronize()
        if offloaded:
            m.offload_stats()
            m.offload_stats_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ext):
            e0.record()
        for i in range(n):
            one(warmup + i)
        st = m.offload_stats() if offloaded else None  # joins the copy streams
        with torch.cuda.stream(ext):
            e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / n, st

    res = p2r.Model(cfg, 1234)
    res.attach_adamw()
    t_res, _ = run(res, False, steps)
    res.close()
    del res
    torch.cuda.empty_cache()
    off = p2r.Model(cfg, 1234, offload=plan, ring_slots=ring)
    off.attach_adamw()
    off.set_grad_accumulation(micro)
    t_off, st = run(off, True, steps)
    off.set_offload_skip_copies(True)
    t_nc, _ = run(off, True, steps)
    off.set_offload_skip_copies(False)
    gran = off.layer_granule_bytes()
    off.close()
    del off
    torch.cuda.empty_cache()
    per = {k: v / steps for k, v in st.items()}
    h2d_b = per["Fn_load"] + per["Bn_load"] + per["opt_load"] + per["grad_load"]
    d2h_b = per["writeback"] + per["grad_offload"]
    t_copy = max(per["h2d_ms"], per["d2h_ms"]) / 1e3
    hidden = 1.0 - max(0.0, t_off - t_nc) / t_copy if t_copy > 0 else 1.0
    T = micro * B * S
    # held-out check of the overlap model (fit on round-1 dense runs): calibrated from
    # this shape's resident step (forward : backward = 1 : 2) and the measured PCIe rates
    P = gran // 18  # (the padded granule)
    h2d_bw = h2d_b / (per["h2d_ms"] / 1e3) if per["h2d_ms"] else 50e9
    d2h_bw = d2h_b / (per["d2h_ms"] / 1e3) if per["d2h_ms"] else 50e9
    tl = t_res / micro / layers
    vec = max(0.0, (per["Fn_load"] / max(1, sum(plan)) - 2 * P) / 4)
    pred = p2r.predict_step_time_overlap([P] * layers, plan, h2d_bw, d2h_bw, tl / 3, 2 * tl / 3,
                                         vector_params=[int(vec)] * layers, fn_master=False,
                                         micro_steps=micro, recompute=True)
    # bytes one SLOW layer must move per optimizer step vs the compute one layer offers
    # per step: the copy / compute ratio that decides how much can hide
    return {"workload": (f"C5 per-rank slice: {layers} Real MoE layers, d=2048, d_ff=4096, 8 local experts top-1, "
                         f"{micro} x {B}x{S} tokens per optimizer step (accumulation), fwd+bwd+AdamW"),
            "placement": plan, "ring_slots": ring, "granule_bytes": gran, "activation_checkpointing": "SLOW layers",
            "step_s": {"resident": round(t_res, 4), "offload": round(t_off, 4), "offload_no_copy": round(t_nc, 4)},
            "tokens_per_s": {"resident": round(T / t_res, 1), "offload": round(T / t_off, 1)},
            "bytes_per_step": {k: per[k] for k in ("Fn_load", "Bn_load", "opt_load", "grad_load", "writeback",
                                                    "grad_offload")},
            "h2d_GBps": round(h2d_b / (per["h2d_ms"] / 1e3) / 1e9, 2) if per["h2d_ms"] else None,
            "d2h_GBps": round(d2h_b / (per["d2h_ms"] / 1e3) / 1e9, 2) if per["d2h_ms"] else None,
            "copy_busy_s": {"h2d": round(per["h2d_ms"] / 1e3, 4), "d2h": round(per["d2h_ms"] / 1e3, 4)},
            "timing": "CUDA events on the model stream (steps) and on the copy streams (busy time)",
            "hidden_fraction": round(hidden, 4),
            "overlap_model": {"predicted_step_s": round(pred, 4), "measured_step_s": round(t_off, 4),
                              "rel_error": round(abs(pred - t_off) / t_off, 4)}}


def main_p2r(args):
    import torch
    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    dist = make_dist(world, local)
    import paper_2110_03888_b200 as p2r

    if args.workload == "c5":
        if world > 1:
            raise SystemExit("c5: per-rank slice, run with --gpus 1 (ranks share nothing)")
        rec = offload_record(p2r, torch, layers=args.layers or 8, steps=args.steps)
        out = {"metric": METRIC, "value": rec["tokens_per_s"]["offload"], "unit": "tokens/s", "n_gpus": 1,
               "steps": args.steps, "warmup": 2, "ms_per_step": round(rec["step_s"]["offload"] * 1e3, 3),
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic", "config": {"workload": rec["workload"], "parallelism": "offload"},
               "offload": rec}
        print(json.dumps(out), flush=True)
        return

    model, B, S, workload, model_flops, graph_ok, par = build_workload(args, p2r, dist, rank, world)
    T = B * S
    model.attach_adamw()
    ext = torch.cuda.ExternalStream(model.stream())
    tok, tgt, mask = lm_batch(B, S, 7 + rank)
    dtok = torch.from_numpy(tok).cuda()
    dtgt = torch.from_numpy(tgt).cuda()
    dmask = torch.from_numpy(mask).cuda()
    loss_dev = torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    denom = float(mask.sum()) * world  # global mask count: summed grads = large-batch mean

    def allreduce():
        if world > 1:
            model.allreduce_grads()  # ncclAllReduce of the replicated grad granules, model stream

    use_graph = graph_ok and not args.no_graph

    def step_device(i, graph=use_graph):
        # one CUDA graph per fwd+bwd step (captured during warm-up); the DP all-reduce
        # and AdamW follow it on the same stream
        model.train_step_device(dtok.data_ptr(), dtgt.data_ptr(), dmask.data_ptr(), B, S, denom,
                                loss_dev=loss_dev.data_ptr(), graph=graph)
        allreduce()
        model.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, i))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for i in range(args.warmup):
        step_device(i)
    barrier()

    # ---- timed region: inputs resident in HBM (activations >> 126 MB L2 per step)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = p2r.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ext):
        e0.record()
    for i in range(args.steps):
        step_device(args.warmup + i)
    with torch.cuda.stream(ext):
        e1.record()
    barrier()
    launches = p2r.launch_count() - launches0
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = T * world / (ms / 1e3)

    # ---- end-to-end through the public host-buffer API
    e2e_steps = max(3, min(args.steps, 10))
    model.train_step(tok, tgt, mask, B, denom)  # untimed: the host path captures its step graph here
    allreduce()
    model.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, args.warmup + args.steps))
    barrier()
    # a pipelined host loop: step i+1 and its optimizer update are enqueued before step i's
    # loss is read back (Model.train_step(wait=False)); every step's inputs still go
    # host -> device and its loss device -> host inside the timed region
    t0 = time.perf_counter()
    prev = None
    for i in range(e2e_steps):
        cur = model.train_step(tok, tgt, mask, B, denom, wait=False)
        allreduce()
        model.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, args.warmup + args.steps + i))
        if prev is not None:
            prev.value()
        prev = cur
    prev.value()
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e = {"value": round(T * world / e2e_s, 1), "unit": "tokens/s",
           "h2d_bytes_per_step": int(tok.nbytes + tgt.nbytes + mask.nbytes), "d2h_bytes_per_step": 4,
           "ms_per_step": round(e2e_s * 1e3, 3)}

    # ---- roofline: the same K steps again in a separate eager pass with every kernel
    # bracketed by CUDA events on the model stream (~2 events per launch, so it is
    # kept out of the `value` region)
    model.profile_reset()
    model.set_profiling(True)
    for i in range(args.steps):
        step_device(args.warmup + args.steps + i, graph=False)  # events need eager launches
    barrier()
    model.set_profiling(False)
    prof = model.profile()

    # ---- roofline of the dominant kernel class
    peaks, peak_src = load_peaks()
    dom = max(prof, key=lambda k: prof[k][1])
    n_l, ms_k, fl, by = prof[dom]
    per_launch_ms = ms_k / max(n_l, 1)
    if fl > 0:
        achieved = fl / (ms_k / 1e3) / 1e12
        peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
        bound, unit = "tensor", "TFLOP/s"
        per_unit = fl / max(n_l, 1)
    else:
        achieved = by / (ms_k / 1e3) / 1e9
        peak = float(peaks["hbm_gbs"])
        bound, unit = "hbm", "GB/s"
        per_unit = by / max(n_l, 1)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath) and args.workload == "c2":
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(dom)
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "peak_source": f"{peak_src} ({'bf16_tflops_sustained' if bound == 'tensor' else 'hbm_gbs'})",
                "timed": "separate eager pass of K steps, CUDA events around every launch on the model stream",
                "launches_per_step": n_l / args.steps, "avg_launch_ms": round(per_launch_ms, 5),
                "algorithmic_per_launch": per_unit}
    breakdown = {k: {"launches": v[0], "ms_per_step": round(v[1] / args.steps, 3),
                     "share": round(v[1] / max(1e-9, sum(x[1] for x in prof.values())), 4),
                     ("tflops" if v[2] > 0 else "gbs"): round((v[2] / 1e12 if v[2] > 0 else v[3] / 1e9) /
                                                              max(v[1] / 1e3, 1e-12), 1)}
                 for k, v in prof.items() if v[0]}
    out = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
           "config": {"workload": workload, "global_batch": B * world, "seq_len": S,
                      "parallelism": par, "l2": "inputs larger than L2 (GBs of activations per step)",
                      "launch": ("one CUDA graph per fwd+bwd step + eager AdamW" if use_graph
                                 else "eager (the expert-parallel exchange's stream flags stay outside graphs)"),
                      "mfu_model_flops_per_token": model_flops},
           "clocks": clk, "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
           "kernels": breakdown,
           "model_tflops": round(model_flops * value / 1e12, 1)}
    model.close()
    del model
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and args.workload == "c2" and not args.no_extras:
        for key, fn in (("moe_ep", moe_ep_record), ("offload", offload_record)):
            try:
                out[key] = fn(p2r, torch)
            except Exception as e:  # noqa: BLE001
                out[key] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0 and world == 1 and args.workload == "c2" and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(ref_procs(args.cpu_procs))
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def relaunch(args):
    """--gpus N > 1 outside torchrun: re-launch this script as N ranks (one per GPU)."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(a))
    if a.impl == "reference":
        main_reference(a)
    else:
        main_p2r(a)
