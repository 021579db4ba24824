"""Switch detector decision logic
through the library's host functions, on scripted loss curves (SPEC's own examples)."""
import numpy as np
import pytest


def test_loss_slope_is_least_squares():
    from paper_2110_03888_b200.switch import loss_slope
    rng = np.random.default_rng(0)
    t = np.sort(rng.uniform(0, 10, 40))
    y = 3.0 - 0.25 * t + rng.normal(0, 0.01, 40)
    assert abs(loss_slope(t, y) - np.polyfit(t, y, 1)[0]) < 1e-12
    assert abs(loss_slope(t, y, 10) - np.polyfit(t[-10:], y[-10:], 1)[0]) < 1e-12


def scripted(step, stage, n, dt=1.0):
    """Loss vs time over a trial starting at `step`: the Pseudo stage decreases at
    -0.01/s until step 500 and plateaus (-0.0005/s) after; Real decreases at -0.004/s."""
    t = np.arange(n + 1) * dt
    if stage == "real":
        return t, 2.0 - 0.004 * t
    rate = 0.01 if step < 500 else 0.0005
    return t, 2.0 - rate * t


def test_detector_fires_after_crossover():
    from paper_2110_03888_b200.switch import SwitchDetector, SwitchPolicy, switch_criterion
    pol = SwitchPolicy(eval_interval_steps=100, trial_budget_steps=20, slope_window=20)
    det = SwitchDetector(pol)
    fired = None
    for step in range(0, 1001, 10):
        if not det.due(step):
            continue
        pt, pl = scripted(step, "pseudo", 20)
        rt, rl = scripted(step, "real", 20)
        fire, ps, rs = switch_criterion(pt, pl, rt, rl, pol)
        if fire and fired is None:
            fired = step
    assert fired == 500  # first evaluation point >= the true crossover, within one interval


def test_detector_never_fires_when_pseudo_steeper():
    from paper_2110_03888_b200.switch import SwitchPolicy, switch_criterion
    pol = SwitchPolicy(100, 20, 20)
    t = np.arange(21.0)
    for step in range(100, 1001, 100):
        fire, ps, rs = switch_criterion(t, 2 - 0.01 * t, t, 2 - 0.004 * t, pol)
        assert not fire and ps < rs


def test_policy_invariants():
    import paper_2110_03888_b200 as p2r
    from paper_2110_03888_b200.switch import SwitchDetector, SwitchPolicy, switch_criterion
    t = np.arange(5.0)
    with pytest.raises(p2r.P2RInvalidArgument, match="trial_budget_steps must not exceed"):
        switch_criterion(t, t, t, t, SwitchPolicy(10, 20, 5))
    with pytest.raises(p2r.P2RInvalidArgument, match="must be positive"):
        SwitchDetector(SwitchPolicy(0, 0, 5)).due(5)
    d = SwitchDetector(SwitchPolicy(500, 50, 50))
    assert [s for s in (0, 250, 500, 750, 1000) if d.due(s)] == [500, 1000]
