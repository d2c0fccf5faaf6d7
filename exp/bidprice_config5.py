"""Config 5 (multi-period, T = 20, shared inventory): the converged SPFOM duals
as bid prices.  Reports how the duals sit against the prices and
runs the bid-price control (sim.bid_price_control) with them and with eta = 0
(offer by r v, no capacity pricing) on the same seeded customer stream."""
import json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2602_22421_b200 import Params, Solver, sim
inst = bench.load_instance("multi", "/tmp/spfom_cache")
s = Solver(inst, Params.converge())
t0 = time.time()
s.step(3000)
eta = s.duals()
r = s.residuals()
s.close()
rel = (inst.price - eta) / inst.price
out = dict(iterations=3000, solve_s=round(time.time() - t0, 2), rel_gap=r["rel_gap"], infeas_rel=r["infeas_rel"],
           eta_eq_r=int(np.sum(np.abs(rel) <= 1e-9)), eta_zero=int(np.sum(eta == 0)), N=int(inst.N),
           max_abs_rel_margin=float(np.abs(rel).max()))
cpp = int(os.environ.get("CPP", "2000"))
for label, e in (("spfom duals", eta), ("eta = 0", np.zeros_like(eta))):
    t = sim.bid_price_control(inst, e, customers_per_period=cpp, seed=7)
    out[label] = dict(revenue=float(t.revenue.sum()), units=float(t.sold.sum()), offers=t.offers,
                      stock_left=float(t.inventory[-1].sum()), min_margin=t.min_margin)
print(json.dumps(out))
