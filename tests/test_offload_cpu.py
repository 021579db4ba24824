"""CPU: the engine's offload planner / cost model (host-only C-ABI) vs the oracle
restatement of SPEC.md:360-377 (exhaustive search for n <= 12) and the SPEC's
known answers (4*W accounting, first-24-of-48, 89 s / 45 s calibration)."""
import os

import numpy as np
import pytest

from oracle import p2r_oracle as O

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2110_03888_b200", "libp2r.so")
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="libp2r.so not built")


def test_planner_uniform_48_offloads_first_24():
    import paper_2110_03888_b200 as p2r
    pl = p2r.plan_offload([100] * 48, 2400, 1.0, 1.0)
    assert pl == [1] * 24 + [0] * 24  # PAPER.md §4.2 "the first 24 layers"
    assert p2r.plan_offload([100] * 48, 4800, 1.0, 1.0) == [0] * 48
    with pytest.raises(p2r.P2RError, match="no feasible plan"):
        p2r.plan_offload([100] * 4, 50, 1.0, 1.0)


@pytest.mark.parametrize("seed", range(6))
def test_planner_matches_exhaustive_oracle(seed):
    import paper_2110_03888_b200 as p2r
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 11))
    lb = [int(x) for x in rng.integers(1, 60, n)]
    budget = int(sum(lb) * rng.uniform(0.3, 0.9))
    mine = p2r.plan_offload(lb, budget, 12.5, 2.0, 0.01)
    ref = O.plan_offload(lb, budget, 12.5, 2.0, 0.01)
    t_mine = p2r.predict_step_time(lb, mine, 12.5, 2.0, 0.01)
    t_ref = O.predict_step_time(lb, ref, 12.5, 2.0, 0.01)
    assert abs(t_mine - t_ref) < 1e-9
    assert sum(b for b, s in zip(lb, mine) if not s) <= budget


def test_cost_model_calibration_89_45():
    """fit on the full-offload point (89 s), predict 24/48 within 10% of 45 s."""
    import paper_2110_03888_b200 as p2r
    compute = 1.0
    bw = 4 * 48 / (89 - compute)
    t_full = p2r.predict_step_time([1] * 48, [1] * 48, bw, compute)
    t_half = p2r.predict_step_time([1] * 48, [1] * 24 + [0] * 24, bw, compute)
    assert abs(t_full - 89) < 1e-9 and abs(t_half - 45) / 45 <= 0.10
