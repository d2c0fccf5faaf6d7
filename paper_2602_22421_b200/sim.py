"""Multi-period bid-price simulation: global optimisation (GO) vs market
segmentation decomposition (MSD) (§5.1.2-5.1.3, Figure 4;
SPEC S:L569-629).

Each batch is a fresh set of customers; the SBLP of the batch (segments =
customers, consideration set = products in stock, capacities = remaining
inventory) is solved with the GPU SPFOM path (`Solver`, the same C ABI as
everything else) to get bid prices eta_j.  The batch's customers stand for
the demand of the remaining horizon: arrival lambda_i = number of remaining
batches (reading c18: the multi-period model assumes the demand distribution
is known in advance, and the bid price is the shadow value of the
remaining capacity, P:L653-660 -- with arrival 1 a single batch never sees
the scarcity of the whole horizon and every bid price is 0).  A customer is shown
the top-`rec_limit` products among {j : r_j - eta_j >= 0}, ranked by
(r_j - eta_j) v_ij, and makes one choice under BAM/MNL (P:L676:
"Customer purchases are simulated under the BAM framework"): product j with
probability v_ij / (v0 + sum_{shown} v_ik).  A sale needs stock (excess demand
is lost).  GO solves one SBLP per batch; MSD splits the batch round-robin into
`segments` groups, each solving its own SBLP against the full remaining
inventory (segments see no global scarcity), then applies the sales
segment by segment to the shared inventory.

This module is an application of the library (the optimisation runs in the
CUDA kernels); the per-customer choice sampling is host bookkeeping.  The
dual solve is a parameter (`solve`, default: the GPU path through `Solver`),
so the same trace can be replayed with another solver's duals -- the tests
replay it with the CPU oracle's.

`bid_price_control` is the bid-price rule itself (offer j iff
r_j - eta_j >= 0) applied to the customers of a multi-period SBLP instance
(BASELINE config 5: "SPFOM duals used as bid prices") with one shared
inventory.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional

import numpy as np

from .spfom import Params, Solver


@dataclasses.dataclass
class SimConfig:
    batches: int = 100
    customers_per_batch: int = 1000
    products: int = 40
    rec_limit: int = 2
    segments: int = 10                    # MSD only
    price_range: tuple = (1.0, 20.0)      # Figure 4 caption
    inventory_range: tuple = (1.0, 2000.0)
    no_purchase: float = 1.0              # BAM outside-option weight
    iters: int = 1500                     # SPFOM iterations per solve
    seed: int = 0


@dataclasses.dataclass
class SimTrace:
    revenue: np.ndarray                   # [batches]
    sold: np.ndarray                      # [batches, products]
    inventory: np.ndarray                 # [batches + 1, products] (row 0 = initial)
    duals: List[Optional[np.ndarray]]     # per batch: bid prices used (None = no solve), per segment for MSD
    solves: int
    offered: Optional[List] = None        # per batch: product mask of what was recommended (per segment for MSD)

    @property
    def cumulative_revenue(self) -> np.ndarray:
        return np.cumsum(self.revenue)


@dataclasses.dataclass
class _BatchInstance:
    """Minimal instance object for `Solver` (the CSR fields it reads)."""
    seg_ptr: np.ndarray
    prod_idx: np.ndarray
    attract: np.ndarray
    shadow: np.ndarray
    no_purchase: np.ndarray
    arrival: np.ndarray
    price: np.ndarray
    capacity: np.ndarray
    meta: dict = dataclasses.field(default_factory=dict)


def market(cfg: SimConfig):
    """Prices and initial inventories (Figure 4: U[1, 20], U[1, 2000]) and the
    per-batch preference draws (U[0, 1] per customer and product)."""
    rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, 4242]))
    prices = rng.uniform(*cfg.price_range, cfg.products)
    inventory = np.floor(rng.uniform(*cfg.inventory_range, cfg.products))
    prefs = [rng.uniform(0.0, 1.0, (cfg.customers_per_batch, cfg.products)) for _ in range(cfg.batches)]
    return prices, inventory, prefs


def gpu_solve(inst, iters: int) -> np.ndarray:
    """The default dual solve: `iters` SPFOM iterations (converge preset) on the GPU."""
    s = Solver(inst, Params.converge())
    s.step(iters)
    eta = s.duals()
    s.close()
    return eta


def _bid_prices(prefs: np.ndarray, avail: np.ndarray, prices: np.ndarray, inventory: np.ndarray,
                cfg: SimConfig, horizon: int, solve: Callable) -> np.ndarray:
    """SBLP of one customer group (arrival = remaining batches each, reading
    c18; consideration set = `avail`; capacities = remaining inventory) solved
    by `solve(instance, iters)`; returns eta over all products (0 off `avail`)."""
    n, k = prefs.shape[0], int(avail.size)
    seg_ptr = np.arange(n + 1, dtype=np.int64) * k
    prod = np.tile(avail.astype(np.int32), n)
    v = np.maximum(prefs[:, avail].reshape(-1), 1e-9)           # attraction > 0 (U[0,1] draws)
    present = np.zeros(prices.shape[0], dtype=bool)
    present[avail] = True
    inst = _BatchInstance(seg_ptr=seg_ptr, prod_idx=prod, attract=v, shadow=np.zeros_like(v),
                          no_purchase=np.full(n, cfg.no_purchase), arrival=np.full(n, float(horizon)),
                          price=np.asarray(prices, float), capacity=np.asarray(inventory, float),
                          meta=dict(present=present))
    return solve(inst, cfg.iters)


def _recommend(prefs: np.ndarray, avail: np.ndarray, margin: np.ndarray, K: int) -> np.ndarray:
    """Per customer: the top-K products among {j in avail : r_j - eta_j >= 0},
    ranked by (r_j - eta_j) v_ij descending.  Returns a boolean
    [customers, products] offer mask."""
    n, m = prefs.shape
    ok = np.zeros(m, dtype=bool)
    ok[avail] = margin[avail] >= 0.0
    score = np.where(ok[None, :], margin[None, :] * prefs, -np.inf)
    offer = np.zeros((n, m), dtype=bool)
    if ok.sum() == 0:
        return offer
    kk = min(K, int(ok.sum()))
    top = np.argsort(-score, axis=1, kind="stable")[:, :kk]
    rows = np.repeat(np.arange(n), kk)
    offer[rows, top.ravel()] = np.isfinite(score[rows, top.ravel()])
    return offer


def _purchase(prefs: np.ndarray, offer: np.ndarray, inventory: np.ndarray, prices: np.ndarray,
              u: np.ndarray, v0: float):
    """One BAM/MNL choice per customer (in order) from its offer set; uniform
    draws `u` fix the randomness.  Sales need stock; returns (revenue, sold)."""
    n, m = prefs.shape
    w = np.where(offer, prefs, 0.0)
    den = v0 + w.sum(axis=1)
    cum = np.cumsum(w, axis=1) / den[:, None]
    choice = np.where(u[:, None] < cum, np.arange(m)[None, :], m).min(axis=1)   # m = no purchase
    sold = np.zeros(m)
    rev = 0.0
    for i in range(n):
        j = int(choice[i])
        if j < m and inventory[j] - sold[j] >= 1.0:
            sold[j] += 1.0
            rev += prices[j]
    return rev, sold


def _run(cfg: SimConfig, segments: int, solve: Optional[Callable] = None) -> SimTrace:
    solve = solve or gpu_solve
    prices, inv0, prefs_all = market(cfg)
    rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, 777]))
    inventory = inv0.copy()
    B, m = cfg.batches, cfg.products
    revenue, sold = np.zeros(B), np.zeros((B, m))
    inv_trace = np.zeros((B + 1, m))
    inv_trace[0] = inventory
    duals: List[Optional[np.ndarray]] = []
    offered: List = []
    solves = 0
    for b in range(B):
        prefs = prefs_all[b]
        u = rng.uniform(0.0, 1.0, prefs.shape[0])          # choice draws, customer order
        avail = np.flatnonzero(inventory >= 1.0)
        groups = [np.arange(prefs.shape[0])[g::segments] for g in range(segments)]
        batch_duals = []
        offers = []
        for gidx in groups:
            if avail.size <= cfg.rec_limit:
                # few products left: recommend all of them
                offer = np.zeros((gidx.size, m), dtype=bool)
                offer[:, avail] = True
                batch_duals.append(None)
            else:
                eta = _bid_prices(prefs[gidx], avail, prices, inventory, cfg, B - b, solve)
                solves += 1
                batch_duals.append(eta)
                offer = _recommend(prefs[gidx], avail, prices - eta, cfg.rec_limit)
            offers.append(offer)
        # sales: segment by segment on the shared inventory (GO: one group)
        rev_b, sold_b = 0.0, np.zeros(m)
        for gidx, offer in zip(groups, offers):
            r, s = _purchase(prefs[gidx], offer, inventory - sold_b, prices, u[gidx], cfg.no_purchase)
            rev_b += r
            sold_b += s
        inventory = inventory - sold_b
        revenue[b], sold[b] = rev_b, sold_b
        inv_trace[b + 1] = inventory
        duals.append(batch_duals[0] if segments == 1 else batch_duals)
        masks = [o.any(axis=0) for o in offers]
        offered.append(masks[0] if segments == 1 else masks)
    return SimTrace(revenue=revenue, sold=sold, inventory=inv_trace, duals=duals, solves=solves, offered=offered)


def run_go_policy(cfg: SimConfig, solve: Optional[Callable] = None) -> SimTrace:
    """GO: one SBLP per batch over all its customers."""
    return _run(cfg, 1, solve)


def run_msd_policy(cfg: SimConfig, solve: Optional[Callable] = None) -> SimTrace:
    """MSD: `cfg.segments` round-robin groups, each with its own SBLP."""
    return _run(cfg, cfg.segments, solve)


def sales_entropy(sold_total: np.ndarray) -> float:
    """Shannon entropy (bits) of the sales distribution over products (App. B.4)."""
    tot = float(np.sum(sold_total))
    if tot <= 0:
        return 0.0
    p = np.asarray(sold_total, float) / tot
    p = p[p > 0]
    return float(-(p * np.log2(p)).sum())


def mean_opportunity_cost(trace: SimTrace) -> float:
    """Average bid price over the (batch, recommended product) pairs of the
    batches with a solve (the opportunity cost of what was
    offered; per segment for MSD)."""
    vals = []
    for b, d in enumerate(trace.duals):
        ds = d if isinstance(d, list) else [d]
        ms = trace.offered[b] if isinstance(trace.offered[b], list) else [trace.offered[b]]
        for e, mask in zip(ds, ms):
            if e is not None:
                vals.extend(np.asarray(e)[mask].tolist())
    return float(np.mean(vals)) if vals else 0.0


@dataclasses.dataclass
class BidPriceTrace:
    revenue: np.ndarray                   # [periods]
    sold: np.ndarray                      # [periods, products]
    inventory: np.ndarray                 # [periods + 1, products] (row 0 = capacity)
    offers: int                           # customers shown at least one product
    min_margin: float                     # smallest |r_j - eta_j| among offered products (ties)


def bid_price_control(inst, eta: np.ndarray, customers_per_period: int, rec_limit: int = 2,
                      seed: int = 0) -> BidPriceTrace:
    """The bid-price rule on a multi-period instance (reading
    c15 stacking, config 5): the converged duals eta_j price the one shared
    inventory c_j.  In period t, customers arrive from base segment i with
    probability proportional to lambda_{i,t}; a customer is shown the top
    `rec_limit` products of C_i in stock with r_j - eta_j >= 0, ranked by
    (r_j - eta_j) v_ij, and buys under GAM: product j of the
    shown set S with probability v_ij / (v_i0 + sum_S v + sum_{C_i \\ S} w);
    a sale takes one unit of inventory.  Seeded draws; host bookkeeping."""
    T = int((getattr(inst, "meta", None) or {}).get("T", 1) or 1)
    M = int(inst.seg_ptr.shape[0] - 1)
    m = M // T
    nb = int(inst.seg_ptr[m])
    seg_ptr = np.asarray(inst.seg_ptr[: m + 1])
    prod, v = np.asarray(inst.prod_idx[:nb]), np.asarray(inst.attract[:nb])
    w = np.asarray(inst.shadow[:nb]) if getattr(inst, "shadow", None) is not None else np.zeros(nb)
    v0 = np.asarray(inst.no_purchase[:m])
    lam = np.asarray(inst.arrival, float).reshape(T, m)
    r = np.asarray(inst.price, float)
    margin = r - np.asarray(eta, float)
    inventory = np.floor(np.asarray(inst.capacity, float))
    rng = np.random.default_rng(np.random.SeedSequence([seed, 515]))
    revenue, sold = np.zeros(T), np.zeros((T, r.shape[0]))
    inv_trace = np.zeros((T + 1, r.shape[0]))
    inv_trace[0] = inventory
    offers, min_margin = 0, np.inf
    for t in range(T):
        p = lam[t] / lam[t].sum()
        segs = rng.choice(m, size=customers_per_period, p=p)
        u = rng.uniform(0.0, 1.0, customers_per_period)
        for c in range(customers_per_period):
            i = int(segs[c])
            a, b = int(seg_ptr[i]), int(seg_ptr[i + 1])
            js, vi, wi = prod[a:b], v[a:b], w[a:b]
            ok = (margin[js] >= 0.0) & (inventory[js] >= 1.0)
            if not ok.any():
                continue
            score = np.where(ok, margin[js] * vi, -np.inf)
            top = np.argsort(-score, kind="stable")[: min(rec_limit, int(ok.sum()))]
            top = top[np.isfinite(score[top])]
            offers += 1
            min_margin = min(min_margin, float(np.abs(margin[js[top]]).min()))
            shown = np.zeros(b - a, dtype=bool)
            shown[top] = True
            den = v0[i] + vi[shown].sum() + wi[~shown].sum()
            cum = np.cumsum(vi[top]) / den
            k = int(np.searchsorted(cum, u[c], side="right"))
            if k < top.size:
                j = int(js[top[k]])
                inventory[j] -= 1.0
                sold[t, j] += 1.0
                revenue[t] += r[j]
        inv_trace[t + 1] = inventory
    return BidPriceTrace(revenue=revenue, sold=sold, inventory=inv_trace, offers=offers,
                         min_margin=float(min_margin))


def cumulative_revenue_identity(trace: SimTrace, prices: np.ndarray) -> float:
    """|sum of batch revenues - sum_j price_j x units sold|."""
    return abs(float(trace.revenue.sum()) - float(prices @ trace.sold.sum(axis=0)))


if __name__ == "__main__":   # Figure-4 style run: python -m paper_2602_22421_b200.sim [runs]
    import json
    import sys

    runs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    out = []
    for r in range(runs):
        cfg = SimConfig(seed=r)
        go, msd = run_go_policy(cfg), run_msd_policy(cfg)
        out.append(dict(seed=r, go_revenue=float(go.revenue.sum()), msd_revenue=float(msd.revenue.sum()),
                        go_entropy=sales_entropy(go.sold.sum(0)), msd_entropy=sales_entropy(msd.sold.sum(0)),
                        go_opportunity_cost=mean_opportunity_cost(go),
                        msd_opportunity_cost=mean_opportunity_cost(msd),
                        go_revenue_per_batch=go.revenue.round(3).tolist(),
                        msd_revenue_per_batch=msd.revenue.round(3).tolist(),
                        go_sold_per_batch=go.sold.sum(1).tolist(), msd_sold_per_batch=msd.sold.sum(1).tolist()))
        print(json.dumps({k: v for k, v in out[-1].items() if not k.endswith("per_batch")}), flush=True)
    print(json.dumps(dict(runs=runs, mean_go=float(np.mean([o["go_revenue"] for o in out])),
                          mean_msd=float(np.mean([o["msd_revenue"] for o in out])))), flush=True)
