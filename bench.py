#!/usr/bin/env python
"""Training-step benchmark of the Pseudo-to-Real hot path on B200.

Workload (BASELINE.json configs[1], "C2"): pseudo-giant dense GPT block shared
across 24 layers, d=1024, 16 heads, d_ff=4096, seq 1024, batch 8 sequences per
GPU, vocab 260, random-init weights (reference init, seed 1234), synthetic
byte tokens. One step = embed -> 24 x block fwd -> tied head -> masked CE ->
full backward (shared-layer grads accumulated in place) -> [NCCL allreduce of
the shared + embedding grads when N > 1] -> AdamW.

  python bench.py [--gpus N --steps K --warmup W]          # this framework
  python bench.py --impl reference [...]                    # reference CPU arm

Prints ONE JSON line on rank 0. `value` = tokens/s over all ranks with inputs
resident in HBM (CUDA events on the model stream, max over ranks); `e2e` = the
same metric through the public host-buffer API (tokens/targets/mask copied in
from pinned memory, loss read back, every step). `roofline` is computed live
from per-kernel CUDA events in the timed region; `cpu_baseline` times the
compiled reference (oracle/_ref) on the host cores on a bounded sample.
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
def main_p2r(args):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2110_03888_b200 as p2r

    B, S = args.batch, C2["seq_len"]
    T = B * S
    model = p2r.Model(p2r.Config(**C2), 1234)
    model.attach_adamw()
    ext = torch.cuda.ExternalStream(model.stream())
    tok, tgt, mask = lm_batch(B, S, 7 + rank)
    dtok = torch.from_numpy(tok).cuda()
    dtgt = torch.from_numpy(tgt).cuda()
    dmask = torch.from_numpy(mask).cuda()
    loss_dev = torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    denom = float(mask.sum()) * world  # global mask count: summed grads = large-batch mean
    if world > 1:
        # the library's own NCCL communicator (csrc/engine/comm.cpp); torch only ships the id
        uid = [p2r.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        model.comm_init(uid[0])

    def allreduce():
        if world > 1:
            model.allreduce_grads()  # ncclAllReduce of the replicated grad granules, model stream

    use_graph = not args.no_graph

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

    # ---- timed region: inputs resident in HBM (activations ~7 GB/step >> 126 MB L2)
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

    # ---- same K steps again with every kernel bracketed by CUDA events on the
    # model stream (kept out of the `value` region: ~2 events per launch)
    model.profile_reset()
    model.set_profiling(True)
    for i in range(args.steps):
        step_device(args.warmup + args.steps + i, graph=False)  # events need eager launches
    barrier()
    model.set_profiling(False)
    prof = model.profile()

    # ---- end-to-end through the public host-buffer API
    e2e_steps = max(3, min(args.steps, 10))
    model.train_step(tok, tgt, mask, B, denom)  # untimed: the host path captures its step graph here
    allreduce()
    model.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, args.warmup + args.steps))
    barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        model.train_step(tok, tgt, mask, B, denom)
        allreduce()
        model.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, args.warmup + args.steps + i))
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e = {"value": round(T * world / e2e_s, 1), "unit": "tokens/s",
           "h2d_bytes_per_step": int(tok.nbytes + tgt.nbytes + mask.nbytes), "d2h_bytes_per_step": 4,
           "ms_per_step": round(e2e_s * 1e3, 3)}

    # ---- roofline of the dominant kernel class, live from the timed region
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
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(dom)
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": bound, "achieved": round(achieved, 2), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dom,
                "peak_source": f"{peak_src} ({'bf16_tflops_sustained' if bound == 'tensor' else 'hbm_gbs'})",
                "launches_per_step": n_l / args.steps, "avg_launch_ms": round(per_launch_ms, 5),
                "algorithmic_per_launch": per_unit}
    breakdown = {k: {"launches": v[0], "ms_per_step": round(v[1] / args.steps, 3),
                     "share": round(v[1] / max(1e-9, sum(x[1] for x in prof.values())), 4),
                     ("tflops" if v[2] > 0 else "gbs"): round((v[2] / 1e12 if v[2] > 0 else v[3] / 1e9) /
                                                              max(v[1] / 1e3, 1e-12), 1)}
                 for k, v in prof.items() if v[0]}
    model_flops = 3 * (24 * (8 * 1024**2 + 4 * 1024 * 4096 + 2 * S * 1024) + 2 * 1024 * 260)
    out = {"metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
           "config": {"workload": WORKLOAD, "global_batch": B * world, "seq_len": S,
                      "parallelism": f"dp{world}", "l2": "inputs larger than L2 (~7 GB activations per step)",
                      "launch": "one CUDA graph per fwd+bwd step + eager AdamW" if use_graph else "eager",
                      "mfu_model_flops_per_token": model_flops},
           "clocks": clk, "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline,
           "kernels": breakdown,
           "model_tflops": round(model_flops * value / 1e12, 1)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline_sample(ref_procs(args.cpu_procs))
        except Exception as e:  # noqa: BLE001
            out["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                                   "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        main_reference(a)
    else:
        main_p2r(a)
