"""Bid-price simulation (GO vs MSD) on the GPU solver."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    from paper_2602_22421_b200.sim import SimConfig
    base = dict(batches=8, customers_per_batch=120, products=12, rec_limit=2, segments=4,
                inventory_range=(1.0, 60.0), iters=400, seed=3)
    base.update(kw)
    return SimConfig(**base)


def test_trace_invariants_and_determinism():
    from paper_2602_22421_b200 import sim
    cfg = _cfg()
    prices, _inv, _p = sim.market(cfg)
    for run in (sim.run_go_policy, sim.run_msd_policy):
        t1, t2 = run(cfg), run(cfg)
        assert np.array_equal(t1.revenue, t2.revenue) and np.array_equal(t1.sold, t2.sold)   # determinism
        inv = t1.inventory
        assert np.all(inv >= 0.0) and np.all(np.diff(inv, axis=0) <= 0.0)
        assert np.all(t1.sold <= inv[:-1])
        assert sim.cumulative_revenue_identity(t1, prices) <= 1e-8
        assert t1.solves > 0


def test_msd_with_one_segment_is_go():
    """a single segment is the global policy (exact trace)."""
    from paper_2602_22421_b200 import sim
    cfg = _cfg(segments=1)
    a, b = sim.run_go_policy(cfg), sim.run_msd_policy(cfg)
    assert np.array_equal(a.revenue, b.revenue) and np.array_equal(a.sold, b.sold)


def test_ample_inventory_recommends_everything_without_solves():
    """products <= rec_limit -> all recommended, no solve."""
    from paper_2602_22421_b200 import sim
    cfg = _cfg(products=3, rec_limit=5, inventory_range=(1e6, 2e6))
    t = sim.run_go_policy(cfg)
    assert t.solves == 0 and all(d is None for d in t.duals)


def test_scarce_inventory_bid_prices_positive():
    """scarce inventory -> strictly positive mean opportunity cost."""
    from paper_2602_22421_b200 import sim
    t = sim.run_go_policy(_cfg(inventory_range=(1.0, 8.0), batches=3))
    assert sim.mean_opportunity_cost(t) > 0.0
