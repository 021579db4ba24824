"""Gradient-parity contract shared by the step-level GPU tests.

North star: loss <= 1e-3 relative, every parameter gradient <= 1e-2 relative L2
(bf16 in / fp32 accumulate vs the fp32 reference). Where the bf16-in design
itself -- oracle/bf16_emulation.py, the fp32 model with bf16 rounding at exactly
the GPU path's rounding points, run on the SAME inputs -- already lands a tensor
at or above ~1e-2 (the attention Q/K projection gradients of unshared layers at
random init, and single expert tensors at d=2048; oracle/precision_floor.py and
DESIGN.md §4 show no single rounding point is responsible), the bound for that
tensor is 1.25x the design floor: the GPU kernels may add at most 25 % on top
of what bf16 inputs cost by themselves."""
import numpy as np


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


def global_rel(gm, gr, names):
    num = sum(float(np.sum((gm[n].astype(np.float64) - gr[n]) ** 2)) for n in names)
    den = sum(float(np.sum(gr[n].astype(np.float64) ** 2)) for n in names)
    return (num / den) ** 0.5


def design_floor(cfgd, params, tok, tgt, mask, batch, denom, forced=None):
    """Gradients of the bf16-in design emulated on the CPU (same inputs / routing)."""
    from oracle import bf16_emulation as BE
    from oracle import p2r_oracle as O
    _, ge = BE.loss_and_grads(O.Config(**cfgd), params, tok, tgt, mask, batch, denom, forced_selected=forced)
    return ge


def check_grads(gm, gr, ge, names, tag, tol=1e-2, strict=True):
    """gm: GPU, gr: fp32 reference, ge: bf16-design emulation. strict: every parameter
    gradient within tol (the north-star contract); strict=False only for
    configs where the bf16-in design's own floor on the same inputs exceeds tol (deep
    Real dense stacks): there the bound is 1.25x that floor."""
    rows = []
    for n in names:
        if np.linalg.norm(gr[n]) == 0:
            assert np.abs(gm[n]).max() == 0.0, n  # top-1 => the gate gradient is exactly 0
            continue
        rows.append((rel(gm[n], gr[n]), rel(ge[n], gr[n]), n))
    rows.sort(reverse=True)
    g = global_rel(gm, gr, [n for _, _, n in rows])
    print(f"[{tag}] global grad rel-L2 {g:.3e}")
    for e, f, n in rows[:6]:
        print(f"[{tag}]   {n:34s} gpu {e:.3e}  bf16-design floor {f:.3e}")
    assert g <= tol
    for e, f, n in rows:
        assert e <= (tol if strict else max(tol, 1.25 * f)), (n, e, f)
    return rows
