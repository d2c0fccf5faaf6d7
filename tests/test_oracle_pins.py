import dataclasses
"""Pins of the CPU oracle against things other than itself (all CPU, -m "not gpu").

Each test names what fixes the expected value: a printed worked example
(tests/golden/spec_examples.json, cited), brute-force enumeration, a closed
form, an invariant, or an LP solved by a different method.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import lp
from spfom_inputs import Instance, generate
from tests.pins import kkt_certificate, project_bruteforce

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rand_segment(rng, k, mnl=False, scale=1.0):
    v = rng.uniform(0.1, 1.0, k)
    w = np.zeros(k) if mnl else v * rng.uniform(0.0, 0.5, k)
    v0 = rng.uniform(0.5, 2.0)
    lam = rng.uniform(1.0, 10.0)
    z0 = rng.normal() * lam * scale
    z = rng.normal(size=k) * lam * scale * rng.uniform(0.0, 1.0)
    return z0, z, v, w, v0, lam


# ------------------------------------------------------------ projection
@pytest.mark.parametrize("seed", range(4))
def test_projection_matches_active_set_enumeration(seed):
    """Pin (i) of c5: KKT active-set enumeration in the original variables, k <= 6."""
    rng = np.random.default_rng(100 + seed)
    worst = 0.0
    for t in range(150):
        k = int(rng.integers(1, 7))
        z0, z, v, w, v0, lam = rand_segment(rng, k, mnl=(t % 4 == 0), scale=[0.1, 1.0, 10.0][t % 3])
        y0, y, _m, _ = oracle.project(z0, z, v, w, v0, lam)
        b0, by = project_bruteforce(z0, z, v, w, v0, lam)
        worst = max(worst, abs(y0 - b0) / lam, np.abs(y - by).max() / lam)
    assert worst <= 1e-13, worst


def test_projection_identity_on_feasible_points():
    """Pin (ii): z in Y_i => Pi(z) = z (feasible points built as convex
    combinations of assortment vertices, App. A.1)."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        k = int(rng.integers(1, 12))
        _z0, _z, v, w, v0, lam = rand_segment(rng, k)
        vt0 = v0 + w.sum()
        y = np.zeros(k)
        wts = rng.dirichlet(np.ones(4))
        for a in wts:
            S = rng.random(k) < 0.5
            U = lam / (vt0 + (v - w)[S].sum())
            y += a * np.where(S, v * U, 0.0)
        y0 = lam - y.sum()
        p0, p, _m, _ = oracle.project(y0, y, v, w, v0, lam)
        assert abs(p0 - y0) <= 1e-13 * lam and np.abs(p - y).max() <= 1e-13 * lam


def test_projection_k1_closed_form():
    """Pin (iv): for k = 1 the GAM polytope is the segment between (lam, 0) and
    (lam v0/(v0+v), lam v/(v0+v)) (GAM reduces to MNL at k = 1: y/v <= y0/v0),
    so the projection is the closed-form projection onto that segment."""
    rng = np.random.default_rng(11)
    for _ in range(500):
        z0, z, v, w, v0, lam = rand_segment(rng, 1, scale=3.0)
        A = np.array([lam, 0.0])
        Bp = np.array([lam * v0[()] if np.ndim(v0) else lam * v0, lam * v[0]]) / (v0 + v[0])
        d = Bp - A
        tt = np.clip(((np.array([z0, z[0]]) - A) @ d) / (d @ d), 0.0, 1.0)
        ref = A + tt * d
        y0, y, _m, _ = oracle.project(z0, z, v, w, v0, lam)
        assert abs(y0 - ref[0]) <= 1e-13 * lam and abs(y[0] - ref[1]) <= 1e-13 * lam


def test_projection_scaling_and_nonexpansive():
    """Pins (v) Pi_{lam Y1}(z) = lam Pi_{Y1}(z/lam) and (vi) ||Pi(z)-Pi(z')|| <= ||z-z'||."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        k = int(rng.integers(1, 40))
        z0, z, v, w, v0, lam = rand_segment(rng, k)
        y0, y, _m, _ = oracle.project(z0, z, v, w, v0, lam)
        u0, u, _m, _ = oracle.project(z0 / lam, z / lam, v, w, v0, 1.0)
        assert abs(y0 - lam * u0) <= 1e-12 * lam and np.abs(y - lam * u).max() <= 1e-12 * lam
        dz0, dz = rng.normal() * 0.3, rng.normal(size=k) * 0.3
        q0, q, _m, _ = oracle.project(z0 + dz0, z + dz, v, w, v0, lam)
        lhs = np.hypot(q0 - y0, np.linalg.norm(q - y))
        rhs = np.hypot(dz0, np.linalg.norm(dz))
        assert lhs <= rhs * (1 + 1e-12) + 1e-13


@pytest.mark.parametrize("k", [50, 200])
def test_projection_kkt_certificate_large_k(k):
    """Pin at any k: NNLS-recovered multipliers prove the oracle's point is the
    projection (stationarity, feasibility, multiplier signs)."""
    rng = np.random.default_rng(k)
    for t in range(20):
        z0, z, v, w, v0, lam = rand_segment(rng, k, scale=[0.05, 1.0, 20.0][t % 3])
        y0, y, _m, _ = oracle.project(z0, z, v, w, v0, lam)
        stat, primal, mmin = kkt_certificate(z0, z, v, w, v0, lam, y0, y)
        assert stat <= 1e-11 and primal <= 1e-12 and mmin >= -1e-12, (stat, primal, mmin)


def test_projection_theta_limit_is_argmax():
    """Pin (iii): Pi(y + theta g) -> argmax_{Y} g^T y as theta -> inf (unique argmax)."""
    rng = np.random.default_rng(5)
    for _ in range(100):
        k = int(rng.integers(1, 30))
        _z0, _z, v, w, v0, lam = rand_segment(rng, k)
        g = rng.lognormal(3.0, 0.5, k) - rng.uniform(0, 30, k)
        val, a0, ay, margin = oracle.argmax(g, v, w, v0, lam)
        if margin < 1e-3:
            continue
        # beyond a finite theta the projection lands exactly on the argmax vertex
        # (g lies inside that vertex's normal cone); 1e6 * |g| keeps rounding at ~1e-9
        y0, y, _m, _ = oracle.project(lam, 1e6 * g, v, w, v0, lam)
        assert np.abs(y - ay).max() <= 1e-8 * lam and abs(y0 - a0) <= 1e-8 * lam


# ------------------------------------------------------------ argmax
def test_argmax_matches_assortment_enumeration():
    """Pin of c6: max over all 2^k assortments of lam sum_j g_j pi_j(S) (CBLP
    single segment, P:L211-219 with GAM pi), k <= 10."""
    rng = np.random.default_rng(21)
    for t in range(300):
        k = int(rng.integers(1, 11))
        _z0, _z, v, w, v0, lam = rand_segment(rng, k, mnl=(t % 3 == 0))
        g = rng.normal(size=k) * 10
        val, y0, y, _mg = oracle.argmax(g, v, w, v0, lam)
        ref = lp.best_assortment_value(g, v, w, v0, lam)
        assert abs(val - ref) <= 1e-13 * max(1.0, abs(ref))
        # the returned point is feasible and attains the value
        assert abs(y0 + y.sum() - lam) <= 1e-13 * lam
        assert abs(float(g @ y) - val) <= 1e-12 * max(1.0, abs(val))


def test_argmax_tie_example():
    for ex in GOLD["argmax_tie"]:
        val, y0, y, margin = oracle.argmax(ex["g"], ex["v"], ex["w"], ex["v0"], ex["lam"])
        assert val == pytest.approx(ex["value"], abs=1e-15)
        assert np.allclose(y, ex["y"], atol=1e-15) and y0 == pytest.approx(ex["y0"], abs=1e-15)
        assert margin == 0.0


def test_argmax_agrees_with_paper_algorithm_1_golden_section():
    """MNL: the paper's own inner solver (FAST-INNER + golden section)
    converges to the exact argmax value as its tolerance shrinks."""
    rng = np.random.default_rng(9)
    for _ in range(200):
        k = int(rng.integers(1, 20))
        _z0, _z, v, _w, v0, lam = rand_segment(rng, k, mnl=True)
        g = rng.normal(size=k) * 5
        val, *_ = oracle.argmax(g, v, np.zeros(k), v0, lam)
        gv, gy0, gy = oracle.golden(g, v, v0, lam, tol=1e-12)
        assert abs(gv - val) <= 1e-8 * max(1.0, abs(val))
        assert gv <= val + 1e-12 * max(1.0, abs(val))        # golden is a feasible point


# ------------------------------------------------------------ SPEC worked examples
def test_spec_fast_inner_examples():
    for ex in GOLD["fast_inner"]:
        z, y = oracle.fast_inner(ex["g"], ex["v"], ex["v0"], ex["lam"], ex["y0"])
        assert z == pytest.approx(ex["z"], abs=1e-14), ex["cite"]
        assert np.allclose(y, ex["y"], atol=1e-14), ex["cite"]


def test_spec_feasible_bound_examples():
    for ex in GOLD["feasible_bound"]:
        g = np.ones(len(ex["v"]))
        z, _ = oracle.fast_inner(g, ex["v"], ex["v0"], ex["lam"], ex["bound"] * (1 + 1e-12))
        assert np.isfinite(z), ex["cite"]
        z, _ = oracle.fast_inner(g, ex["v"], ex["v0"], ex["lam"], ex["bound"] * (1 - 1e-6))
        assert np.isnan(z), ex["cite"]


def test_spec_golden_examples():
    for ex in GOLD["golden"]:
        # value at a kink converges linearly in the bracket width
        val, y0, _y = oracle.golden(ex["g"], ex["v"], ex["v0"], ex["lam"], tol=1e-9)
        assert val == pytest.approx(ex["value"], abs=1e-6), ex["cite"]


def test_spec_dual_step_examples():
    for ex in GOLD["dual_step"]:
        out = oracle.dual_step([ex["eta"]], [ex["s"]], [ex["s"]], [ex["c"]], [ex["tau"]], ex["mu"], 0.0)
        assert out[0] == pytest.approx(ex["out"], abs=1e-15), ex["cite"]


def test_dual_step_extrapolation_hand_example():
    """st = s + omega (s - s_prev) = 2 + 1*(2 - 1.5) = 2.5 -> 0.2 - 0.1 (1 - 2.5) = 0.35."""
    out = oracle.dual_step([0.2], [2.0], [1.5], [1.0], [0.1], 0.0, 1.0)
    assert out[0] == pytest.approx(0.35, abs=1e-15)


def _inst(seg_ptr, prod, v, w, v0, lam, r, c):
    N = len(r)
    prod = np.asarray(prod, dtype=np.int32)
    return Instance("hand", np.asarray(seg_ptr, dtype=np.int64), prod, np.asarray(v, float),
                    np.asarray(w, float), np.asarray(v0, float), np.asarray(lam, float),
                    np.asarray(r, float), np.asarray(c, float),
                    np.bincount(prod, minlength=N) > 0, {})


def test_spec_compute_R():
    ex = GOLD["compute_R"][0]
    inst = _inst([0, 2, 4], [0, 1, 0, 1], ex["v_rows"][0] + ex["v_rows"][1], [0] * 4, [1, 1], [1, 1],
                 ex["r"], [1, 1])
    R = oracle.compute_R(inst)
    assert R == pytest.approx(ex["R"], abs=1e-15) and 1 / (2 * R) == pytest.approx(ex["mu"])


@pytest.mark.parametrize("ex", GOLD["sblp_1x1"], ids=lambda e: e["cite"])
def test_spec_sblp_1x1(ex):
    """n = m = 1 SBLP optimum: dense simplex, HiGHS and SPFOM (converge preset) agree with S:L458-460."""
    inst = _inst([0, 1], [0], [ex["v"]], [0.0], [ex["v0"]], [ex["lam"]], [ex["r"]], [ex["c"]])
    assert lp.sblp_dense(inst)[0] == pytest.approx(ex["obj"], abs=1e-12)
    assert lp.sblp_highs(inst)[0] == pytest.approx(ex["obj"], abs=1e-9)
    S = oracle.OracleSolver(inst, theta=1.0, tau=0.9, tau_mode=1, mu=0.0, extrapolation=1.0)
    S.run(3000)
    assert S.residuals()["primal_obj"] == pytest.approx(ex["obj"], abs=1e-9)
    assert S.y[0] == pytest.approx(ex["y"], abs=1e-9)


def test_spec_choice_probabilities():
    for ex in GOLD["choice_prob"]:
        pi = lp.gam_choice_prob(np.array(ex["v"]), np.array(ex["w"]), ex["v0"], ex["S"])
        assert np.allclose(pi, ex["pi"], atol=1e-15), ex["cite"]


# ------------------------------------------------------------ LP references
def test_tiny_sblp_equals_cblp_enumeration():
    """c3/c12: dense simplex SBLP = HiGHS SBLP = CBLP enumeration LP (dense and
    HiGHS), capacitated and uncapacitated; uncapacitated also = sum of per-segment
    best assortments."""
    for seed in (1, 11, 12):
        inst = generate("tiny", seed=seed)
        for unc in (False, True):
            a = lp.sblp_dense(inst, uncapacitated=unc)[0]
            b = lp.sblp_highs(inst, uncapacitated=unc)[0]
            c = lp.cblp_lp(inst, uncapacitated=unc)
            d = lp.cblp_lp(inst, uncapacitated=unc, solver="highs")
            assert max(abs(a - b), abs(a - c), abs(a - d)) <= 1e-9 * abs(a)
            if unc:
                e = sum(lp.best_assortment_value(inst.price[inst.prod_idx[inst.row(i)]],
                                                 inst.attract[inst.row(i)], inst.shadow[inst.row(i)],
                                                 inst.no_purchase[i], inst.arrival[i])
                        for i in range(inst.m))
                assert abs(a - e) <= 1e-9 * abs(a)


# ------------------------------------------------------------ the iteration
def _check_state_invariants(S, inst):
    res = S.residuals()
    assert res["balance_rel_max"] <= 1e-13 and res["scale_rel_max"] <= 1e-13 and res["neg_max"] == 0.0
    assert (S.eta >= 0).all()
    fresh = np.bincount(inst.prod_idx, weights=S.y, minlength=inst.N)
    assert np.abs(fresh - S.s).max() <= 1e-12 * max(1.0, np.abs(fresh).max())


def test_oracle_iterates_stay_feasible_and_usage_consistent():
    inst = generate("small", m=300, N=200, k=30)
    S = oracle.OracleSolver(inst)
    for _ in range(30):
        S.step()
        _check_state_invariants(S, inst)


@pytest.mark.parametrize("seed", [1, 11, 12, 13, 14])
def test_converge_preset_reaches_tiny_lp_optimum(seed):
    """c8/c11: converge preset (theta=1, tau_j = 0.9/n_j, omega_x = 1, mu = 0, full
    sweep), 2000 iterations, vs the dense-simplex P*: <= 1e-9 relative, infeasible <= 1e-9."""
    inst = generate("tiny", seed=seed)
    Pstar = lp.sblp_dense(inst)[0]
    S = oracle.OracleSolver(inst)
    S.run(2000)
    res = S.residuals()
    assert abs(res["primal_obj"] - Pstar) <= 1e-9 * Pstar
    assert res["infeas_rel"] <= 1e-9
    assert res["cert_lower"] <= Pstar * (1 + 1e-12) and Pstar <= res["cert_upper"] * (1 + 1e-12)


def test_dual_bound_is_weak_duality_upper_bound():
    """D(eta) >= P* for any eta >= 0 (A.3), here random eta on tiny."""
    inst = generate("tiny")
    Pstar = lp.sblp_dense(inst)[0]
    S = oracle.OracleSolver(inst)
    rng = np.random.default_rng(0)
    for _ in range(50):
        eta = rng.uniform(0, 10, inst.N) * (rng.random(inst.N) < 0.7)
        assert S.residuals(eta=eta)["dual_obj"] >= Pstar - 1e-12 * Pstar


def test_sampled_mode_touches_only_block_rows_and_tracks_usage():
    """c2/c7: with a sampled block only the block's rows change, s is the
    incremental stale-inclusive sum and equals a fresh recompute."""
    from spfom_inputs import block_sequence
    inst = generate("small", m=400, N=150, k=20)
    blocks = block_sequence(inst.m, 37, 40, seed=5)
    S = oracle.OracleSolver(inst, theta=np.inf, tau=0.1, tau_mode=0, mu=0.5, extrapolation=0.0)
    for t in range(40):
        y_before = S.y.copy()
        S.step(blocks[t])
        changed_rows = set(np.searchsorted(inst.seg_ptr, np.flatnonzero(S.y != y_before), side="right") - 1)
        assert changed_rows <= set(blocks[t].tolist())
        _check_state_invariants(S, inst)


def test_paper_preset_first_iteration_closed_form():
    """theta = inf from eta = 0: every row is its unconstrained best assortment
    (enumeration), then eta = max(0, -tau (c - s)) (Alg. 2)."""
    inst = generate("tiny")
    S = oracle.OracleSolver(inst, theta=np.inf, tau=0.1, tau_mode=0, mu=0.0, extrapolation=0.0)
    S.step()
    for i in range(inst.m):
        sl = inst.row(i)
        ref = lp.best_assortment_value(inst.price[inst.prod_idx[sl]], inst.attract[sl], inst.shadow[sl],
                                       inst.no_purchase[i], inst.arrival[i])
        assert float(inst.price[inst.prod_idx[sl]] @ S.y[sl]) == pytest.approx(ref, rel=1e-13)
    s = np.bincount(inst.prod_idx, weights=S.y, minlength=inst.N)
    assert np.allclose(S.eta, np.maximum(0.0, -0.1 * (inst.capacity - s)), rtol=0, atol=1e-14)


def test_averaging_is_uniform_mean_of_iterates():
    """a8 (reading c9): the running average equals the mean of the stored iterates."""
    inst = generate("small", m=100, N=60, k=10)
    A = oracle.OracleSolver(inst, averaging=True)
    B = oracle.OracleSolver(inst)
    ys, etas = [], []
    for _ in range(25):
        A.step()
        B.step()
        ys.append(B.y.copy())
        etas.append(B.eta.copy())
    assert np.abs(A.ybar - np.mean(ys, axis=0)).max() <= 1e-13 * max(1, np.abs(A.ybar).max())
    assert np.abs(A.etabar - np.mean(etas, axis=0)).max() <= 1e-13 * max(1, np.abs(A.etabar).max())


def test_shard_primitives_compose_to_iterate():
    """primal_shard + dual_apply on the whole instance is oracle_iterate's full
    sweep (the primitives used by the sharded emulation), bit for bit."""
    inst = generate("small", m=200, N=120, k=(5, 40))
    A = oracle.OracleSolver(inst)
    B = oracle.OracleSolver(inst)
    for _ in range(15):
        A.step()
        B.dual_apply(B.primal_shard())
        assert np.array_equal(A.y, B.y) and np.array_equal(A.eta, B.eta) and np.array_equal(A.s, B.s)


def test_oracle_reaches_small_lp_optimum():
    """Converge preset on the BASELINE small config (seed 2), 3000 iterations, vs
    the HiGHS optimum stored by tests/golden/make_lp_optima.py (oracle-only script)."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lp_optima.json")))["small"]
    inst = generate("small")
    S = oracle.OracleSolver(inst)
    S.run(3000)
    res = S.residuals()
    assert abs(res["primal_obj"] - gold["Pstar"]) <= 1e-6 * gold["Pstar"]
    assert res["infeas_rel"] <= 1e-6
    assert res["cert_lower"] <= gold["Pstar"] * (1 + 1e-9) <= res["cert_upper"] * (1 + 2e-9)


def test_multi_period_T1_and_stacking():
    """c15: T = 1 multi-period == single period; stacked P* == sum over the
    period LP with shared capacities solved directly (dense simplex on the
    stacked rows == HiGHS on the same)."""
    a = generate("multi", m=3, N=5, k=3, T=1)
    b = generate("multi", m=3, N=5, k=3, T=2)
    assert b.m == 2 * a.m and np.array_equal(b.prod_idx[: a.nnz], a.prod_idx)
    assert lp.sblp_dense(b)[0] == pytest.approx(lp.sblp_highs(b)[0], rel=1e-9)


# ------------------------------------------------------------ SBLP -> CBLP recovery
def test_recover_spec_worked_example():
    """m = 1, lambda = 1, w0 = w1 = 1 (MNL), y = (0.75, 0.25) ->
    alpha({0}) = 0.5, alpha({0,1}) = 0.5 (paper letters: w = attraction)."""
    order, alpha = oracle.recover(0.75, [0.25], [1.0], [0.0], 1.0, 1.0, [0])
    assert list(order) == [0] and np.allclose(alpha, [0.5, 0.5], atol=1e-15)


def test_recover_degenerate_rows():
    rng = np.random.default_rng(5)
    k = 6
    v = rng.uniform(0.1, 1, k)
    w = v * rng.uniform(0, 0.5, k)
    v0, lam = 1.3, 2.0
    # all mass on the no-purchase option: alpha(S_0) = 1
    _o, a = oracle.recover(lam, np.zeros(k), v, w, v0, lam, np.arange(k))
    assert abs(a[0] - 1.0) <= 1e-15 and np.all(a[1:] == 0.0)
    # the full-assortment vertex: every ratio equals U -> one atom on S_k
    vt0 = v0 + w.sum()
    U = lam / (vt0 + (v - w).sum())
    y = v * U
    y0 = lam - y.sum()
    _o, a = oracle.recover(y0, y, v, w, v0, lam, np.arange(k))
    assert abs(a[k] - 1.0) <= 1e-12 and np.all(np.abs(a[:k]) <= 1e-12)


@pytest.mark.parametrize("seed", range(6))
def test_recover_reproduces_feasible_rows(seed):
    """The recovered nested-assortment policy reproduces the row it came from
    under the GAM choice model: lambda sum_l alpha_l pi_j(S_l) = y_j,
    the same for the no-purchase share, sum alpha = 1, alpha >= 0, and the
    revenue identity -- checked on rows the oracle projection makes
    feasible, including capped (tied) entries and zeros."""
    rng = np.random.default_rng(100 + seed)
    for _ in range(60):
        k = int(rng.integers(1, 9))
        v = rng.uniform(0.1, 1, k)
        w = v * rng.uniform(0, 0.5, k)
        v0, lam = rng.uniform(0.5, 2), rng.uniform(1, 10)
        z = rng.normal(0, 3, k)
        y0, y, _m, _it = oracle.project(rng.uniform(0, lam), z, v, w, v0, lam)
        prod = rng.permutation(50)[:k].astype(np.int32)
        order, alpha = oracle.recover(y0, y, v, w, v0, lam, prod)
        assert sorted(order) == list(range(k))
        u = y / v
        assert all(u[order[i]] >= u[order[i + 1]] for i in range(k - 1))
        assert abs(alpha.sum() - 1.0) <= 1e-12 and alpha.min() >= -1e-14
        q0, q = oracle.policy_probabilities(order, alpha, v, w, v0)
        assert np.abs(lam * q - y).max() <= 1e-12 * lam and abs(lam * q0 - y0) <= 1e-12 * lam
        r = rng.uniform(1, 10, k)
        rev = lam * sum(alpha[l] * sum(r[j] * v[j] for j in order[:l]) /
                        (v0 + sum(v[j] if j in set(order[:l]) else w[j] for j in range(k))) for l in range(k + 1))
        assert abs(rev - float(r @ y)) <= 1e-11 * max(1.0, float(r @ y))


def test_recover_tie_order_by_product_index():
    """Equal ratios are ordered by ascending product id."""
    v = np.array([0.5, 0.25, 1.0])
    y = v * 0.2                      # all ratios equal
    order, _a = oracle.recover(1.0, y, v, np.zeros(3), 1.0, 1.0 + y.sum(), np.array([7, 3, 5], np.int32))
    assert list(order) == [1, 2, 0]


# ------------------------------------------------------------ bundles / NRM
def test_bundle_identity_incidence_reduces_to_the_base():
    """Reduction law: Bt = I, c_l = c_j gives the base
    trajectory bit for bit."""
    from spfom_inputs import with_bundles
    inst = generate("small", m=200, N=120, k=(5, 40))
    a = oracle.OracleSolver(inst)
    b = oracle.OracleSolver(with_bundles(inst, identity=True))
    for _ in range(30):
        a.step()
        b.step()
    assert np.array_equal(a.y, b.y) and np.array_equal(a.y0, b.y0) and np.array_equal(a.eta, b.eta)
    assert a.residuals() == b.residuals()


def test_bundle_effective_coefficients_spec_example():
    """bundle 1 = {resources 1, 2}, eta = (0.3, 0.2), r_1 = 1 -> 0.5;
    eta = 0 -> r."""
    from spfom_inputs import with_bundles
    inst = generate("tiny")
    b = with_bundles(inst, identity=True)
    ptr = np.array([0, 2] + [2 + j for j in range(1, inst.N)], dtype=np.int64)
    res = np.array([0, 1] + [j % 2 for j in range(1, inst.N)], dtype=np.int32)
    b = dataclasses.replace(b, num_resources=2, bundle_ptr=ptr, bundle_res=res, resource_capacity=np.ones(2),
                            price=np.concatenate([[1.0], inst.price[1:]]))
    S = oracle.OracleSolver(b)
    g = S.prices(np.array([0.3, 0.2]))
    assert abs(g[0] - 0.5) <= 1e-15
    assert np.array_equal(S.prices(np.zeros(2)), b.price)


def test_bundle_converges_to_the_generalized_lp_optimum():
    """The bundle SPFOM (per-resource tau_l = 0.9 / n_l, converge preset) heads
    to the Eq. 33 LP optimum (HiGHS on the sparse U-auxiliary form with resource
    rows; coupled resources converge slower than the base SBLP: 1e-4 after 8000
    iterations), and every iterate brackets it: (1 - alpha) P <= P* <= D(eta)
    (weak duality of the bundle Lagrangian)."""
    from oracle import lp
    from spfom_inputs import with_bundles
    inst = with_bundles(generate("small", m=300, N=60, k=(5, 20)), L=24, seed=3, rho=0.5)
    Pstar, _y, _y0 = lp.sblp_highs(inst)
    S = oracle.OracleSolver(inst)
    for it in range(8):
        for _ in range(1000):
            S.step()
        r = S.residuals()
        assert r["cert_lower"] <= Pstar * (1 + 1e-12) and Pstar <= r["cert_upper"] * (1 + 1e-12), (it, r, Pstar)
    assert abs(r["primal_obj"] - Pstar) <= 1e-4 * Pstar, (r["primal_obj"], Pstar)
    assert r["infeas_rel"] <= 1e-3


def test_bundle_infinite_capacity_keeps_resource_duals_zero():
    """non-binding resources -> eta = 0."""
    from spfom_inputs import with_bundles
    inst = with_bundles(generate("small", m=100, N=40, k=(5, 20)), L=10, seed=1)
    inst = dataclasses.replace(inst, resource_capacity=np.full(10, 1e12))
    S = oracle.OracleSolver(inst)
    for _ in range(20):
        S.step()
    assert np.all(S.eta == 0.0)


# ------------------------------------------------------------ bid-price simulation helpers
def test_sales_entropy_examples():
    from paper_2602_22421_b200.sim import sales_entropy
    assert abs(sales_entropy(np.array([3, 3, 3, 3])) - 2.0) <= 1e-15
    assert sales_entropy(np.array([0, 7, 0])) == 0.0
    assert abs(sales_entropy(np.array([2, 1, 1])) - 1.5) <= 1e-15
    assert sales_entropy(np.zeros(5)) == 0.0


# ------------------------------------------------------------ step sizes and residual pins
def _dense_A(inst):
    """The SBLP capacity matrix written out densely: row j (product), one
    column per variable y_ij, coefficient 1 where segment i considers j
    (Eq. 8; A = [M | I])."""
    A = np.zeros((inst.N, inst.nnz))
    A[inst.prod_idx, np.arange(inst.nnz)] = 1.0
    return A


def test_tau_is_the_inverse_squared_row_norm_of_A():
    """c8 (Pock-Chambolle diagonal preconditioning): tau_j = tau0 / ||A_j||^2
    with A the dense capacity matrix (||A_j||^2 = n_j, P:L1111-1125's rho
    corrected); tau_mode 0 is the scalar tau."""
    inst = generate("small", m=120, N=60, k=(5, 30))
    A = _dense_A(inst)
    row2 = (A * A).sum(axis=1)
    tau1 = oracle.OracleSolver(inst, tau=0.9, tau_mode=1).tau_j
    want = np.where(row2 > 0, 0.9 / np.maximum(row2, 1.0), 0.9)
    assert np.array_equal(tau1, want)
    tau0 = oracle.OracleSolver(inst, tau=0.1, tau_mode=0).tau_j
    assert np.all(tau0 == 0.1)


def test_bundle_tau_is_the_row_sum_of_Bt_A():
    """c17: per resource tau_l = tau0 / sum_col |(Bt A)_l,col|, Bt the dense
    bundle -> resource incidence (Eq. 33)."""
    from spfom_inputs import with_bundles
    inst = with_bundles(generate("small", m=120, N=60, k=(5, 30)), L=25, seed=3)
    Bt = np.zeros((inst.num_resources, inst.N))
    for j in range(inst.N):
        Bt[inst.bundle_res[inst.bundle_ptr[j]:inst.bundle_ptr[j + 1]], j] = 1.0
    rows = np.abs(Bt @ _dense_A(inst)).sum(axis=1)
    tau = oracle.OracleSolver(inst, tau=0.9, tau_mode=1).tau_j
    assert np.allclose(tau, np.where(rows > 0, 0.9 / np.maximum(rows, 1.0), 0.9), rtol=0, atol=0)


@pytest.mark.parametrize("seed", [1, 11])
def test_complementary_slackness_vanishes_at_the_lp_optimum(seed):
    """c11 compl_slack = sum_j eta_j |c_j - s_j| / (1 + |P|): at a primal-dual
    optimal pair of the LP every positive dual has a binding capacity (KKT
    complementary slackness), so the converged iterate gives ~0, while an
    arbitrary positive eta with slack capacities gives a positive value."""
    inst = generate("tiny", seed=seed)
    S = oracle.OracleSolver(inst)
    S.run(2000)
    res = S.residuals()
    assert res["compl_slack"] <= 1e-9 and res["rel_gap"] <= 1e-9
    s = _dense_A(inst) @ S.y
    eta = np.ones(inst.N)
    slack = S.residuals(eta=eta)["compl_slack"]
    assert slack == pytest.approx(np.abs(inst.capacity - s).sum() / (1 + abs(res["primal_obj"])), rel=1e-12)
    assert slack > 0.0


def test_l2_infeasibility_is_bracketed_by_the_max_infeasibility():
    """c11 infeas_rel_l2 = ||(s - c)^+||_2 / (1 + ||c||_2) against infeas_abs =
    ||(s - c)^+||_inf: inf-norm <= 2-norm <= sqrt(N) inf-norm; both 0 exactly
    when every capacity holds."""
    inst = generate("small", m=200, N=80, k=(5, 30))
    S = oracle.OracleSolver(inst)
    S.run(3)                               # early: capacities violated
    r = S.residuals()
    cn = np.linalg.norm(inst.capacity[inst.present])
    lo, hi = r["infeas_abs"] / (1 + cn), np.sqrt(inst.N) * r["infeas_abs"] / (1 + cn)
    assert r["infeas_abs"] > 0 and lo * (1 - 1e-12) <= r["infeas_rel_l2"] <= hi * (1 + 1e-12)
    y0 = np.asarray(inst.arrival, float).copy()
    r0 = S.residuals(eta=np.zeros(inst.N), y=np.zeros(inst.nnz), y0=y0)    # y = 0: s = 0 <= c
    assert r0["infeas_abs"] == 0.0 and r0["infeas_rel_l2"] == 0.0
