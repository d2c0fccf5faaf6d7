"""Seeded instance and block-sequence generators (BASELINE.json configs).

Recipe:

* Consideration sets C_i: successive sampling without replacement -- draw
  products i.i.d. from the popularity law p and keep the first k_i distinct
  ones.  p is uniform ("small") or Zipf(s) over popularity ranks, the rank ->
  product-id map being a seeded permutation (so product ids carry no
  popularity order; the CUDA path relabels, the oracle never does).
* v_ij ~ U(0.1, 1) (attraction), w_ij = u_ij * v_ij with u_ij ~ U(0, 0.5)
  drawn per (i, j) (GAM shadow attraction; tiny: u = 0.3), v_i0 ~ U(0.5, 2)
  (tiny: 1), r_j ~ LogNormal(3, 0.5) (tiny: U(1, 10)), lambda_i ~ U(1, 10)
  (tiny: U(1, 5); multi-period: U(0.5, 5) per (i, t)).
* c_j = rho * d_j with the full-offer demand
  d_j = sum_{i : j in C_i} lambda_i v_ij / (v_i0 + sum_{k in C_i} v_ik)
  (the GAM purchase probability when the whole consideration set is offered;
  BASELINE.json's "uncapacitated demand", reading c1).  Products no segment
  considers (n_j = 0) get c_j = 1 and present[j] = False.
* Streams: numpy PCG64, SeedSequence(seed).spawn(4) ->
  [structure, weights, prices/lambda, blocks].

The module computes no part of the SPFOM iteration; it is shared by the
oracle tests and the CUDA path only as a source of inputs.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

# name -> recipe.  k: int (fixed) or (lo, hi) inclusive uniform integer range,
# or "all" (every segment considers every product).
CONFIGS = {
    "tiny": dict(seed=1, m=4, N=6, k="all", pop="uniform", zipf_s=None,
                 v0=("const", 1.0), shadow=("frac", 0.3), price=("uniform", 1.0, 10.0),
                 arrival=("uniform", 1.0, 5.0), rho=0.5, T=1),
    "small": dict(seed=2, m=1000, N=500, k=50, pop="uniform", zipf_s=None,
                  v0=("uniform", 0.5, 2.0), shadow=("uvar", 0.0, 0.5), price=("lognormal", 3.0, 0.5),
                  arrival=("uniform", 1.0, 10.0), rho=0.5, T=1),
    "medium": dict(seed=3, m=100_000, N=10_000, k=(20, 200), pop="zipf", zipf_s=1.1,
                   v0=("uniform", 0.5, 2.0), shadow=("uvar", 0.0, 0.5), price=("lognormal", 3.0, 0.5),
                   arrival=("uniform", 1.0, 10.0), rho=0.4, T=1),
    "huge": dict(seed=4, m=1_000_000, N=100_000, k=50, pop="zipf", zipf_s=1.1,
                 v0=("uniform", 0.5, 2.0), shadow=("uvar", 0.0, 0.5), price=("lognormal", 3.0, 0.5),
                 arrival=("uniform", 1.0, 10.0), rho=0.3, T=1),
    # multi-period: m is the per-period segment count; stacked period-major.
    "multi": dict(seed=5, m=100_000, N=20_000, k=50, pop="zipf", zipf_s=1.1,
                  v0=("uniform", 0.5, 2.0), shadow=("uvar", 0.0, 0.5), price=("lognormal", 3.0, 0.5),
                  arrival=("uniform", 0.5, 5.0), rho=0.3, T=20),
}


def config_spec(name: str, **overrides) -> dict:
    spec = dict(CONFIGS[name])
    for key, val in overrides.items():
        if key not in spec:
            raise KeyError(f"unknown config key {key!r}")
        spec[key] = val
    return spec


@dataclasses.dataclass
class Instance:
    """CSR segment x consideration-set instance, original product order.

    BASELINE naming: m segments i, N products j; v = attraction, w = shadow.
    """

    name: str
    seg_ptr: np.ndarray      # int64 [m+1]
    prod_idx: np.ndarray     # int32 [nnz], strictly increasing within a row
    attract: np.ndarray      # f64 [nnz]  v_ij > 0
    shadow: np.ndarray       # f64 [nnz]  0 <= w_ij < v_ij
    no_purchase: np.ndarray  # f64 [m]    v_i0 > 0
    arrival: np.ndarray      # f64 [m]    lambda_i > 0
    price: np.ndarray        # f64 [N]    r_j
    capacity: np.ndarray     # f64 [N]    c_j
    present: np.ndarray      # bool [N]   n_j > 0
    meta: dict
    # bundles / NRM (Eq. 33): products are bundles over L base resources
    num_resources: int = 0
    bundle_ptr: Optional[np.ndarray] = None          # int64 [N+1] CSR: resources of bundle j
    bundle_res: Optional[np.ndarray] = None          # int32 [nnz_B], strictly increasing per bundle
    resource_capacity: Optional[np.ndarray] = None   # f64 [L]

    @property
    def m(self) -> int:
        return int(self.seg_ptr.shape[0] - 1)

    @property
    def N(self) -> int:
        return int(self.price.shape[0])

    @property
    def nnz(self) -> int:
        return int(self.prod_idx.shape[0])

    def row(self, i: int) -> slice:
        return slice(int(self.seg_ptr[i]), int(self.seg_ptr[i + 1]))

    def segment_slice(self, lo: int, hi: int) -> "Instance":
        """Segments [lo, hi) with the same product space (a rank's shard)."""
        a, b = int(self.seg_ptr[lo]), int(self.seg_ptr[hi])
        return Instance(
            name=f"{self.name}[{lo}:{hi}]",
            seg_ptr=(self.seg_ptr[lo:hi + 1] - a).astype(np.int64),
            prod_idx=self.prod_idx[a:b], attract=self.attract[a:b], shadow=self.shadow[a:b],
            no_purchase=self.no_purchase[lo:hi], arrival=self.arrival[lo:hi],
            price=self.price, capacity=self.capacity, present=self.present,
            meta=dict(self.meta, shard=(lo, hi)), num_resources=self.num_resources, bundle_ptr=self.bundle_ptr,
            bundle_res=self.bundle_res, resource_capacity=self.resource_capacity)


def _draw(rng: np.random.Generator, kind: tuple, size) -> np.ndarray:
    if kind[0] == "uniform":
        return rng.uniform(kind[1], kind[2], size)
    if kind[0] == "lognormal":
        return rng.lognormal(kind[1], kind[2], size)
    if kind[0] == "const":
        return np.full(size, float(kind[1]))
    raise ValueError(kind)


def _row_lengths(rng: np.random.Generator, spec: dict) -> np.ndarray:
    m, N, k = spec["m"], spec["N"], spec["k"]
    if k == "all":
        return np.full(m, N, dtype=np.int64)
    if isinstance(k, (tuple, list)):
        lo, hi = int(k[0]), int(k[1])
        return rng.integers(lo, hi + 1, size=m).astype(np.int64)
    return np.full(m, int(k), dtype=np.int64)


def _successive_sample(rng: np.random.Generator, cdf: np.ndarray, ks: np.ndarray) -> np.ndarray:
    """For every row draw ks[i] distinct ids (popularity-rank space) by
    successive sampling: i.i.d. draws from the law whose CDF is `cdf`, keeping
    first occurrences in draw order until ks[i] are collected.  Returns the
    concatenated ids, row-major, unsorted within a row."""
    m = ks.shape[0]
    out = np.empty(int(ks.sum()), dtype=np.int64)
    offs = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(ks, out=offs[1:])
    todo = np.arange(m)
    mult = 3
    while todo.size:
        kmax = int(ks[todo].max())
        D = mult * kmax + 64
        chunk = max(1, 20_000_000 // D)
        failed = []
        for c0 in range(0, todo.size, chunk):
            rows = todo[c0:c0 + chunk]
            kr = ks[rows]
            draws = np.searchsorted(cdf, rng.random((rows.size, D)), side="right")
            draws = np.minimum(draws, cdf.size - 1)
            order = np.argsort(draws, axis=1, kind="stable")
            sd = np.take_along_axis(draws, order, 1)
            first_sorted = np.ones(sd.shape, dtype=bool)
            first_sorted[:, 1:] = sd[:, 1:] != sd[:, :-1]
            first = np.empty_like(first_sorted)
            np.put_along_axis(first, order, first_sorted, 1)
            cnt = np.cumsum(first, axis=1)
            ok = cnt[:, -1] >= kr
            keep = first & (cnt <= kr[:, None]) & ok[:, None]
            vals = draws[keep]
            okrows = rows[ok]
            # rows are contiguous in `vals` in row order
            starts = np.zeros(okrows.size + 1, dtype=np.int64)
            np.cumsum(ks[okrows], out=starts[1:])
            dst = np.repeat(offs[okrows], ks[okrows]) + (np.arange(vals.size) - np.repeat(starts[:-1], ks[okrows]))
            out[dst] = vals
            failed.append(rows[~ok])
        todo = np.concatenate(failed) if failed else np.zeros(0, dtype=np.int64)
        mult *= 2
    return out


def _structure(rng: np.random.Generator, spec: dict):
    m, N = spec["m"], spec["N"]
    ks = _row_lengths(rng, spec)
    if np.any(ks > N) or np.any(ks < 1):
        raise ValueError("consideration-set size must be in [1, N]")
    seg_ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(ks, out=seg_ptr[1:])
    if spec["k"] == "all":
        prod = np.tile(np.arange(N, dtype=np.int64), m)
        return seg_ptr, prod.astype(np.int32)
    if spec["pop"] == "zipf":
        ranks = np.arange(1, N + 1, dtype=np.float64)
        p = ranks ** (-float(spec["zipf_s"]))
    else:
        p = np.ones(N)
    cdf = np.cumsum(p / p.sum())
    cdf[-1] = 1.0
    perm = rng.permutation(N)                   # popularity rank -> product id
    ids = perm[_successive_sample(rng, cdf, ks)]
    rows = np.repeat(np.arange(m, dtype=np.int64), ks)
    order = np.lexsort((ids, rows))
    prod = ids[order].astype(np.int32)
    return seg_ptr, prod


def _full_offer_demand(seg_ptr, prod, v, v0, lam, N) -> np.ndarray:
    ks = np.diff(seg_ptr)
    nonempty = ks > 0
    rowsum = np.zeros(v0.shape[0])
    rowsum[nonempty] = np.add.reduceat(v, seg_ptr[:-1][nonempty])
    scale = lam / (v0 + rowsum)
    return np.bincount(prod, weights=v * np.repeat(scale, ks), minlength=N)


def generate(name: str, seed: Optional[int] = None, **overrides) -> Instance:
    """Instance for BASELINE config `name` (tiny/small/medium/huge/multi).

    `overrides` rescale a recipe for parity tests (e.g. m=2000, N=400) while
    keeping its distributions; `seed` defaults to the config's seed."""
    spec = config_spec(name, **overrides)
    if seed is None:
        seed = spec["seed"]
    s_struct, s_weights, s_prices, _s_blocks = np.random.SeedSequence(seed).spawn(4)
    r_struct = np.random.Generator(np.random.PCG64(s_struct))
    r_w = np.random.Generator(np.random.PCG64(s_weights))
    r_p = np.random.Generator(np.random.PCG64(s_prices))

    seg_ptr, prod = _structure(r_struct, spec)
    m, N, nnz = spec["m"], spec["N"], int(prod.shape[0])
    v = r_w.uniform(0.1, 1.0, nnz)
    sh = spec["shadow"]
    if sh[0] == "frac":
        w = sh[1] * v
    else:
        w = r_w.uniform(sh[1], sh[2], nnz) * v
    v0 = _draw(r_w, spec["v0"], m)
    r = _draw(r_p, spec["price"], N)
    T = int(spec["T"])
    lam = _draw(r_p, spec["arrival"], (T, m))

    counts = np.bincount(prod, minlength=N)
    present = counts > 0
    demand = np.zeros(N)
    for t in range(T):
        demand += _full_offer_demand(seg_ptr, prod, v, v0, lam[t], N)
    cap = np.where(present, spec["rho"] * demand, 1.0)

    meta = dict(config=name, seed=int(seed), spec={k: (list(x) if isinstance(x, tuple) else x)
                                                   for k, x in spec.items()}, T=T)
    if T == 1:
        return Instance(name=name, seg_ptr=seg_ptr, prod_idx=prod, attract=v, shadow=w,
                        no_purchase=v0, arrival=lam[0], price=r, capacity=cap,
                        present=present, meta=meta)
    base = Instance(name=name + "-base", seg_ptr=seg_ptr, prod_idx=prod, attract=v, shadow=w,
                    no_purchase=v0, arrival=lam[0], price=r, capacity=cap, present=present,
                    meta=dict(meta, T=1))
    return stack_periods(base, lam, cap, name=name, meta=meta)


def stack_periods(base: Instance, lam_tm: np.ndarray, capacity: np.ndarray,
                  name: str = "stacked", meta: Optional[dict] = None) -> Instance:
    """Period-major stacking (SPEC stack_periods; reading c15): segment
    t*m + i is base segment i in period t, with arrival lam_tm[t, i]; the
    consideration sets and v/w/v0 are shared across periods and all periods
    share one inventory c_j."""
    T = int(lam_tm.shape[0])
    m, nnz = base.m, base.nnz
    seg_ptr = np.concatenate(
        [[0], (base.seg_ptr[1:][None, :] + np.arange(T)[:, None] * nnz).ravel()]).astype(np.int64)
    return Instance(
        name=name, seg_ptr=seg_ptr,
        prod_idx=np.tile(base.prod_idx, T), attract=np.tile(base.attract, T),
        shadow=np.tile(base.shadow, T), no_purchase=np.tile(base.no_purchase, T),
        arrival=np.ascontiguousarray(lam_tm.reshape(T * m)), price=base.price,
        capacity=np.asarray(capacity, dtype=np.float64), present=base.present,
        meta=dict(meta or {}, T=T, m_per_period=m))


def period_slice(inst: Instance, lo: int, hi: int) -> Instance:
    """Base segments [lo, hi) of a period-major stacked multi-period instance,
    in every period (a rank's shard when whole segments -- all T periods --
    stay on one rank); still stacked period-major."""
    T = int(inst.meta.get("T", 1))
    m = int(inst.meta.get("m_per_period", inst.m // T))
    rows = [inst.segment_slice(t * m + lo, t * m + hi) for t in range(T)]
    nb = rows[0].nnz
    seg_ptr = np.concatenate([[0]] + [r.seg_ptr[1:] + t * nb for t, r in enumerate(rows)]).astype(np.int64)
    cat = lambda name: np.concatenate([getattr(r, name) for r in rows])
    return Instance(name=f"{inst.name}[base {lo}:{hi}]", seg_ptr=seg_ptr, prod_idx=cat("prod_idx"),
                    attract=cat("attract"), shadow=cat("shadow"), no_purchase=cat("no_purchase"),
                    arrival=cat("arrival"), price=inst.price, capacity=inst.capacity, present=inst.present,
                    meta=dict(inst.meta, T=T, m_per_period=hi - lo, shard=(lo, hi)), num_resources=inst.num_resources,
                    bundle_ptr=inst.bundle_ptr, bundle_res=inst.bundle_res, resource_capacity=inst.resource_capacity)


def with_bundles(inst: Instance, L: Optional[int] = None, seed: int = 0, rho: float = 0.4,
                 identity: bool = False) -> Instance:
    """NRM bundling instance (SPEC BundleInstance S:L44-47): the
    products of `inst` become bundles over L base resources.  Recipe: bundle j
    consumes resource perm(j) mod L and, with probability 1/2, one more distinct
    uniform resource (so every bundle consumes 1 or 2 resources, every resource
    is used when L <= N); c_l = rho x sum_{j : l in B_j} d_j with d_j the
    full-offer demand of bundle j (reading c1 applied per resource).
    identity=True: L = N, B = I, c_l = c_j (the reduction law)."""
    N = inst.N
    if identity:
        ptr = np.arange(N + 1, dtype=np.int64)
        res = np.arange(N, dtype=np.int32)
        return dataclasses.replace(inst, num_resources=N, bundle_ptr=ptr, bundle_res=res,
                                   resource_capacity=np.array(inst.capacity, dtype=np.float64),
                                   meta=dict(inst.meta, bundles="identity"))
    L = int(L if L is not None else max(1, N // 2))
    rng = np.random.default_rng(np.random.SeedSequence([seed, 7717]))
    perm = rng.permutation(N)
    rows = []
    for j in range(N):
        a = int(perm[j] % L)
        r = {a}
        if L > 1 and rng.random() < 0.5:
            b = int(rng.integers(0, L - 1))
            r.add(b if b < a else b + 1)
        rows.append(sorted(r))
    ptr = np.zeros(N + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(r) for r in rows])
    res = np.concatenate([np.asarray(r, dtype=np.int32) for r in rows]) if N else np.zeros(0, np.int32)
    T = int(inst.meta.get("T", 1))
    m1 = int(inst.meta.get("m_per_period", inst.m // T))
    d = np.zeros(N)
    for t in range(T):      # full-offer demand of every bundle, summed over periods
        sub = inst.segment_slice(t * m1, (t + 1) * m1) if T > 1 else inst
        d += _full_offer_demand(sub.seg_ptr, sub.prod_idx, sub.attract, sub.no_purchase, sub.arrival, N)
    cres = np.zeros(L)
    for j in range(N):
        for l in rows[j]:
            cres[l] += d[j]
    cres = rho * cres
    cres[cres <= 0] = 1.0
    return dataclasses.replace(inst, num_resources=L, bundle_ptr=ptr, bundle_res=res, resource_capacity=cres,
                               meta=dict(inst.meta, bundles=dict(L=L, seed=seed, rho=rho)))


def block_sequence(m: int, B: int, iters: int, seed: int) -> np.ndarray:
    """Pre-generated sampled blocks I_t ("Randomly generate a subset of
    customers ... with size B"; reading c2): int32 [iters][B], each row B
    distinct segment ids drawn uniformly without replacement, sorted."""
    if not 1 <= B <= m:
        raise ValueError("need 1 <= B <= m")
    ss = np.random.SeedSequence(seed).spawn(4)[3]
    rng = np.random.Generator(np.random.PCG64(ss))
    out = np.empty((iters, B), dtype=np.int32)
    for t in range(iters):
        out[t] = np.sort(rng.choice(m, B, replace=False))
    return out
