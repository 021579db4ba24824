"""Pseudo -> Real switch detector.

Decision logic lives in libp2r (csrc/engine/switch.cpp); this module binds it
and drives one evaluation on a live Pseudo model through the checkpoint API:

    det = SwitchDetector(SwitchPolicy(eval_interval_steps=500, trial_budget_steps=50, slope_window=50))
    if det.due(step):
        res = det.evaluate(model, step_fn, eval_fn, "/tmp/snapshot.p2rckpt")
        if res["fire"]: ...switch to the Real stage (delink_checkpoint / Model.delinked)...

step_fn(m) trains `m` for one step; eval_fn(m) returns its evaluation loss.
"""
import ctypes
import time
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib


class SwitchPolicyC(ctypes.Structure):
    _fields_ = [("eval_interval_steps", ctypes.c_int), ("trial_budget_steps", ctypes.c_int),
                ("slope_window", ctypes.c_int)]


@dataclass
class SwitchPolicy:
    """SPEC.md:255-259; defaults are the SPEC design decision (500 / 50 / 50)."""
    eval_interval_steps: int = 500
    trial_budget_steps: int = 50
    slope_window: int = 50

    def c(self) -> SwitchPolicyC:
        return SwitchPolicyC(self.eval_interval_steps, self.trial_budget_steps, self.slope_window)


def _declare():
    L = lib()
    dp = ctypes.POINTER(ctypes.c_double)
    L.p2r_loss_slope.argtypes = [dp, dp, ctypes.c_int, ctypes.c_int, dp]
    L.p2r_switch_criterion.argtypes = [dp, dp, ctypes.c_int, dp, dp, ctypes.c_int, ctypes.POINTER(SwitchPolicyC),
                                       ctypes.POINTER(ctypes.c_int), dp, dp]
    L.p2r_switch_evaluation_due.argtypes = [ctypes.POINTER(SwitchPolicyC), ctypes.c_int64, ctypes.POINTER(ctypes.c_int)]
    return L


def _d(a):
    a = np.ascontiguousarray(a, np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def loss_slope(time_s, loss, window: int = 0) -> float:
    """Least-squares d loss / d time over the last `window` points (all if <= 0)."""
    L = _declare()
    (t, tp), (l, lp) = _d(time_s), _d(loss)
    out = ctypes.c_double()
    check(L.p2r_loss_slope(tp, lp, len(t), window, ctypes.byref(out)))
    return out.value


def switch_criterion(pseudo_t, pseudo_loss, real_t, real_loss, policy: SwitchPolicy):
    """(fire, pseudo_slope, real_slope): fire when Real decreases loss faster."""
    L = _declare()
    (pt, ptp), (pl, plp), (rt, rtp), (rl, rlp) = _d(pseudo_t), _d(pseudo_loss), _d(real_t), _d(real_loss)
    fire, ps, rs = ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    check(L.p2r_switch_criterion(ptp, plp, len(pt), rtp, rlp, len(rt), ctypes.byref(policy.c()), ctypes.byref(fire),
                                 ctypes.byref(ps), ctypes.byref(rs)))
    return bool(fire.value), ps.value, rs.value


class SwitchDetector:
    def __init__(self, policy: SwitchPolicy, clock=time.perf_counter):
        self.policy = policy
        self.clock = clock
        self.history = []  # one record per evaluation

    def due(self, step: int) -> bool:
        L = _declare()
        out = ctypes.c_int()
        check(L.p2r_switch_evaluation_due(ctypes.byref(self.policy.c()), int(step), ctypes.byref(out)))
        return bool(out.value)

    def evaluate(self, model, step_fn, eval_fn, snapshot_path: str, step: int = 0) -> dict:
        """One SPEC detect_switch evaluation on the live Pseudo `model`:
        snapshot -> delink -> Real trial (trial_budget_steps) -> revert -> Pseudo
        continuation for the same wall time -> compare loss slopes. The Real trial
        is discarded; the Pseudo model ends up continued from the snapshot."""
        model.save_checkpoint(snapshot_path, stage="PSEUDO", global_step=step)
        real = model.delinked()
        t0 = self.clock()
        rt, rl = [0.0], [float(eval_fn(real))]
        for _ in range(self.policy.trial_budget_steps):
            step_fn(real)
            rt.append(self.clock() - t0)
            rl.append(float(eval_fn(real)))
        budget = rt[-1]
        real.close()
        model.load_checkpoint(snapshot_path)  # revert: bit-equal to the snapshot
        t0 = self.clock()
        pt, pl = [0.0], [float(eval_fn(model))]
        while True:
            step_fn(model)
            pt.append(self.clock() - t0)
            pl.append(float(eval_fn(model)))
            if pt[-1] >= budget:
                break
        fire, ps, rs = switch_criterion(pt, pl, rt, rl, self.policy)
        rec = {"step": step, "fire": fire, "pseudo_slope": ps, "real_slope": rs, "trial_s": budget,
               "pseudo_steps": len(pt) - 1}
        self.history.append(rec)
        return rec
