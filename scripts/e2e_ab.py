"""Interleaved A/B in one process: device-resident graph steps (bench `value`) vs the
pipelined host-API steps (bench `e2e`), 10 steps per block, CUDA events on the model stream."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2110_03888_b200 as p2r  # noqa: E402

m = p2r.Model(p2r.Config(**bench.C2), 1234)
m.attach_adamw()
B, S = 8, 1024
tok, tgt, mask = bench.lm_batch(B, S, 7)
denom = float(mask.sum())
ext = torch.cuda.ExternalStream(m.stream())
dt, dg, dm = (torch.from_numpy(x).cuda() for x in (tok, tgt, mask))
loss_dev = torch.zeros(1, device="cuda")


def dev_block():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ext):
        e0.record()
    for _ in range(10):
        m.train_step_device(dt.data_ptr(), dg.data_ptr(), dm.data_ptr(), B, S, denom, loss_dev=loss_dev.data_ptr(),
                            graph=True)
        m.adamw_step(1e-4)
    with torch.cuda.stream(ext):
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


def host_block():
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ext):
        e0.record()
    t0 = time.perf_counter()
    prev = None
    for _ in range(10):
        cur = m.train_step(tok, tgt, mask, B, denom, wait=False)
        m.adamw_step(1e-4)
        if prev is not None:
            prev.value()
        prev = cur
    prev.value()
    wall = (time.perf_counter() - t0) / 10 * 1e3
    with torch.cuda.stream(ext):
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10, wall


for _ in range(2):
    dev_block()
    host_block()
for r in range(3):
    d = dev_block()
    h, w = host_block()
    print(f"round {r}: device graph {d:.3f} ms/step | host pipelined {h:.3f} ms/step (wall {w:.3f})")
