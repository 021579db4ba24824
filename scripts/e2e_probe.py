"""Where the end-to-end (host API) step spends its time beyond the device step:
times train_step / adamw_step host calls and the device step for C2."""
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
for i in range(4):
    m.train_step(tok, tgt, mask, B, denom)
    m.adamw_step(1e-4)
torch.cuda.synchronize()
ts, ta = [], []
t0 = time.perf_counter()
for i in range(10):
    a = time.perf_counter()
    m.train_step(tok, tgt, mask, B, denom)
    b = time.perf_counter()
    m.adamw_step(p2r.lr_at(2e-4, 0.01, 1000, i))
    c = time.perf_counter()
    ts.append(b - a)
    ta.append(c - b)
torch.cuda.synchronize()
tt = (time.perf_counter() - t0) / 10
print(f"e2e step {tt*1e3:.3f} ms: train_step call {np.mean(ts)*1e3:.3f} ms, adamw call {np.mean(ta)*1e3:.3f} ms")
ext = torch.cuda.ExternalStream(m.stream())
dt, dg, dm = (torch.from_numpy(x).cuda() for x in (tok, tgt, mask))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(3):
    m.train_step_device(dt.data_ptr(), dg.data_ptr(), dm.data_ptr(), B, S, denom, graph=True)
    m.adamw_step(1e-4)
torch.cuda.synchronize()
with torch.cuda.stream(ext):
    e0.record()
for i in range(10):
    m.train_step_device(dt.data_ptr(), dg.data_ptr(), dm.data_ptr(), B, S, denom, graph=True)
    m.adamw_step(1e-4)
with torch.cuda.stream(ext):
    e1.record()
torch.cuda.synchronize()
print(f"device step {e0.elapsed_time(e1)/10:.3f} ms")

# pipelined host loop (bench's e2e): per-step device time vs the gaps between steps,
# from events recorded on the model stream between the host calls
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
prev = None
t0 = time.perf_counter()
for i in range(10):
    with torch.cuda.stream(ext):
        evs[i][0].record()
    cur = m.train_step(tok, tgt, mask, B, denom, wait=False)
    m.adamw_step(1e-4)
    with torch.cuda.stream(ext):
        evs[i][1].record()
    if prev is not None:
        prev.value()
    prev = cur
prev.value()
tt = (time.perf_counter() - t0) / 10
torch.cuda.synchronize()
busy = [a.elapsed_time(b) for a, b in evs]
gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(9)]
print(f"pipelined e2e {tt*1e3:.3f} ms/step wall; device per step {np.mean(busy):.3f} ms "
      f"(min {min(busy):.3f}), gap between steps {np.mean(gaps)*1e3:.1f} us (max {max(gaps)*1e3:.1f})")
