"""GPU parity: the CUDA path through the C ABI vs the CPU oracle (-m gpu).

Tolerances (north_star / SURVEY §8(c) c13): per-iterate rel-inf <= 1e-10 for
the first 100 iterations; final objective within 1e-6 of the LP optimum;
primal infeasibility <= 1e-6.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import lp
from spfom_inputs import Instance, block_sequence, generate
from tests.parity import TOL_ITER, lockstep, oracle_kwargs, rel_inf

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "lp_optima.json")


def _params(**kw):
    from paper_2602_22421_b200 import Params
    return Params(**kw)


def _paper(**kw):
    from paper_2602_22421_b200 import Params
    return Params.paper(**kw)


def _assert_ok(worst):
    assert "first_bad_iter" not in worst and max(worst[k] for k in ("y", "y0", "eta", "s")) <= TOL_ITER, worst


# ------------------------------------------------------------ per-iterate parity
@pytest.mark.parametrize("name,kw", [
    ("tiny", {}),
    ("small", {}),
    ("medium", dict(m=2000, N=1500, k=(20, 200))),          # four length bins, Zipf head
    ("multi", dict(m=400, N=300, k=50, T=3)),               # stacked periods, shared inventory
])
@pytest.mark.parametrize("exec_mode", [0, 1])               # auto (persistent small regime here) / graph
def test_converge_preset_lockstep_100(name, kw, exec_mode):
    inst = generate(name, **kw)
    worst, gpu, _ = lockstep(inst, _params(exec_mode=exec_mode), 100)
    gpu.close()
    _assert_ok(worst)


@pytest.mark.parametrize("preset,B", [("converge", None), ("converge", 300), ("paper", 40)])
def test_exec_modes_agree(preset, B):
    """The persistent cooperative small-regime kernel (exec_mode 2: whole
    iterations per launch, grid barriers) and the per-iteration graph
    (exec_mode 1) compute the same iterates."""
    from paper_2602_22421_b200 import Params, Solver
    inst = generate("medium", m=1500, N=1200, k=(20, 200))
    blocks = None if B is None else block_sequence(inst.m, B, 16, 3)
    mk = (lambda **kw: Params.converge(blocks=blocks, **kw)) if preset == "converge" else \
         (lambda **kw: Params.paper(blocks=blocks, mu=0.5, **kw))
    a, b = Solver(inst, mk(exec_mode=2)), Solver(inst, mk(exec_mode=1))
    a.step(25)
    b.step(25)
    assert a.iteration == b.iteration == 25
    ya, y0a = a.primal()
    yb, y0b = b.primal()
    lam = float(inst.arrival.max())
    assert rel_inf(ya, yb, lam) <= 1e-12 and rel_inf(y0a, y0b, lam) <= 1e-12
    assert rel_inf(a.duals(), b.duals(), float(inst.price.max())) <= 1e-12
    a.close()
    b.close()


def _ragged_instance(ks, N=1100, seed=0):
    rng = np.random.default_rng(seed)
    rows = [np.sort(rng.choice(N, k, replace=False)) for k in ks]
    seg_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    prod = np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32)
    nnz = prod.shape[0]
    v = rng.uniform(0.1, 1.0, nnz)
    w = v * rng.uniform(0.0, 0.5, nnz)
    m = len(ks)
    v0 = rng.uniform(0.5, 2.0, m)
    lam = rng.uniform(1.0, 10.0, m)
    r = rng.lognormal(3.0, 0.5, N)
    cnt = np.bincount(prod, minlength=N)
    d = np.zeros(N)
    for i in range(m):
        sl = slice(seg_ptr[i], seg_ptr[i + 1])
        d += np.bincount(prod[sl], weights=lam[i] * v[sl] / (v0[i] + v[sl].sum()), minlength=N)
    c = np.where(cnt > 0, 0.4 * d, 1.0)
    return Instance("ragged", seg_ptr, prod, v, w, v0, lam, r, c, cnt > 0, {})


def test_ragged_lengths_cross_every_bin_and_pad():
    """Edge cases: k = 0 (empty consideration set), 1, pad widths 1..3, every
    bin boundary (16/32/52/104/208/512/1024 entries) and the old ones."""
    ks = [0, 1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 51, 52, 53, 63, 64, 65, 103, 104, 105, 127, 128, 129,
          200, 207, 208, 209, 255, 256, 257, 300, 511, 512, 513, 1000, 1024, 0, 6, 50] * 3
    inst = _ragged_instance(ks)
    worst, gpu, cpu = lockstep(inst, _params(), 60)
    gpu.close()
    _assert_ok(worst)


def _degenerate_instance(m, N, ks, seed=0):
    rng = np.random.default_rng(seed)
    rows = [np.sort(rng.choice(N, k, replace=False)) for k in ks]
    seg_ptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    prod = np.concatenate(rows).astype(np.int32) if sum(ks) else np.zeros(0, np.int32)
    nnz = prod.shape[0]
    v = rng.uniform(0.1, 1.0, nnz)
    w = v * rng.uniform(0.0, 0.5, nnz)
    cnt = np.bincount(prod, minlength=N)
    return Instance("degenerate", seg_ptr, prod, v, w, rng.uniform(0.5, 2.0, m), rng.uniform(1.0, 10.0, m),
                    rng.lognormal(3.0, 0.5, N), np.where(cnt > 0, 0.3, 1.0), cnt > 0, {})


@pytest.mark.parametrize("exec_mode", [0, 1])
@pytest.mark.parametrize("case", ["no segments", "every row empty", "one segment, one product", "B = 1"])
def test_degenerate_instances(case, exec_mode):
    """The method's degenerate cases through every execution mode: m = 0 (no
    primal work: the dual step alone, eta stays 0 on the absent products'
    slack capacity); rows with k = 0 only (y_i0 = lambda_i, A y = 0); a
    single segment offered a single product (the k = 1 closed form of the
    projection); sampled blocks of one segment."""
    blocks = None
    if case == "no segments":
        inst = _degenerate_instance(0, 3, [])
    elif case == "every row empty":
        inst = _degenerate_instance(5, 4, [0] * 5)
    elif case == "one segment, one product":
        inst = _degenerate_instance(1, 1, [1])
    else:
        inst = _degenerate_instance(7, 6, [3, 0, 6, 1, 2, 5, 4])
        blocks = block_sequence(inst.m, 1, 16, 5)
    worst, gpu, _ = lockstep(inst, _params(exec_mode=exec_mode, blocks=blocks), 40, blocks=blocks)
    gpu.close()
    _assert_ok(worst)


@pytest.mark.parametrize("preset,k", [("converge", (49, 52)), ("paper", (49, 52)), ("converge", (33, 52)),
                                      ("converge", 50)])
def test_entry_mapped_bin_lockstep(preset, k):
    """Rows of 33..52 entries (9..13 quads; the k = 50 configs have 13) run on
    the full-sweep stream kernel's entry mapping (bin E = 13: 4 lanes x 13
    entries).  k in 49..52 or k = 50: every row has exactly 13
    quads (the uniform-row fast path; the last round of the bin is partial);
    33..52: ragged rows (per-entry bounds).  24000 segments give every warp >= 2
    rounds, so the throughput mapping runs, not the wide latency one."""
    inst = generate("huge", m=24000 + 5, N=3000, k=k)
    p = _params(exec_mode=1) if preset == "converge" else _paper(mu=0.5, exec_mode=1)
    worst, gpu, _ = lockstep(inst, p, 100, check_every=5, check_first=5)
    gpu.close()
    _assert_ok(worst)


@pytest.mark.parametrize("preset", ["paper", "converge"])
@pytest.mark.parametrize("case", ["uniform E13", "ragged E13", "medium bins", "medium wide", "every bin"])
def test_sampled_stream_lockstep(case, preset):
    """Sampled blocks through the stream kernels' row gather (SAMP
    instantiations, exec_mode 1 = graph): the block's rows of each bin are
    gathered into the slots by 16-B copies and the usage scatter adds
    y_new - y_old.  uniform E13: k = 50 (13 quads, the UNI path) with
    N = 20000 > the shared/spread head, so the tail reductions run; ragged:
    33..52 entries (per-entry bounds); medium bins: blocks big enough for the
    throughput mappings of the G = 4 / 8 / 16 entry-mapped bins; medium wide:
    small blocks (the wide latency mappings).  Per-iterate rel-inf <= 1e-10 vs
    the oracle run on the same blocks."""
    if case == "uniform E13":
        inst, B, it = generate("huge", m=48005, N=20000, k=50), 24001, 60
    elif case == "ragged E13":
        inst, B, it = generate("huge", m=48005, N=3000, k=(33, 52)), 24001, 60
    elif case == "medium bins":
        inst, B, it = generate("medium", m=100000, N=6000, k=(20, 200)), 60000, 30
    elif case == "medium wide":
        inst, B, it = generate("medium", m=8000, N=3000, k=(20, 200)), 1500, 100
    else:                       # k = 0 rows, pads, every bin boundary (the longest rows: list kernel)
        ks = [0, 1, 3, 4, 5, 16, 17, 32, 33, 52, 53, 104, 105, 208, 209, 512, 513, 1000] * 40
        inst, B, it = _ragged_instance(ks, N=1100, seed=5), 400, 60
    blocks = block_sequence(inst.m, B, 16, seed=9)
    p = _params(blocks=blocks, exec_mode=1) if preset == "converge" else _paper(mu=0.5, blocks=blocks, exec_mode=1)
    worst, gpu, _ = lockstep(inst, p, it, blocks=blocks, check_every=5, check_first=3)
    assert not gpu.info()["persistent"]
    gpu.close()
    _assert_ok(worst)


def test_mnl_special_case_lockstep():
    """omega = 0 (MNL) is the GAM special case."""
    inst = generate("small", m=500, N=300, k=(10, 80))
    inst.shadow[:] = 0.0
    worst, gpu, _ = lockstep(inst, _params(), 60)
    gpu.close()
    _assert_ok(worst)


def test_theta_variants_lockstep():
    inst = generate("small", m=600, N=300, k=(10, 70))
    for theta in (0.05, 0.3, 5.0):
        worst, gpu, _ = lockstep(inst, _params(theta=theta, tau=0.9 / max(theta, 1.0)), 40)
        gpu.close()
        _assert_ok(worst)


def test_paper_preset_sampled_lockstep_100():
    """Alg. 2 literal: theta = inf (exact inner argmax), scalar tau = 0.1,
    Eq. 17 with mu = 0.5, sampled blocks of B = 100, no extrapolation."""
    inst = generate("small")
    blocks = block_sequence(inst.m, 100, 100, seed=7)
    worst, gpu, cpu = lockstep(inst, _paper(mu=0.5, blocks=blocks), 100, blocks=blocks)
    gpu.close()
    _assert_ok(worst)


def test_paper_preset_full_sweep_lockstep():
    inst = generate("small", m=800, N=400, k=(10, 90))
    worst, gpu, _ = lockstep(inst, _paper(mu=0.0), 100)
    gpu.close()
    _assert_ok(worst)


def test_sampled_finite_theta_with_refresh():
    inst = generate("medium", m=1500, N=600, k=(20, 120))
    blocks = block_sequence(inst.m, 257, 13, seed=3)
    worst, gpu, _ = lockstep(inst, _params(blocks=blocks, refresh_every=7), 60, blocks=blocks)
    gpu.close()
    _assert_ok(worst)


def test_averaging_parity():
    inst = generate("small", m=500, N=250, k=(5, 60))
    p = _params(averaging=True)
    worst, gpu, cpu = lockstep(inst, p, 50)
    _assert_ok(worst)
    yb, y0b, eb = gpu.averages()
    gpu.close()
    lam, rmax = float(inst.arrival.max()), float(inst.price.max())
    assert rel_inf(yb, cpu.ybar, lam) <= TOL_ITER and rel_inf(y0b, cpu.y0bar, lam) <= TOL_ITER
    assert rel_inf(eb, cpu.etabar, rmax) <= TOL_ITER


def test_residuals_match_oracle():
    inst = generate("small")
    worst, gpu, cpu = lockstep(inst, _params(), 50, check_every=50)
    _assert_ok(worst)
    rg = gpu.residuals()
    ro = cpu.residuals()
    gpu.close()
    for k in ("primal_obj", "dual_obj", "cert_lower", "cert_upper"):
        assert abs(rg[k] - ro[k]) <= 1e-10 * abs(ro[k]), (k, rg[k], ro[k])
    for k in ("infeas_abs", "infeas_rel", "infeas_rel_l2", "alpha", "compl_slack"):
        assert abs(rg[k] - ro[k]) <= 1e-10 * max(1.0, abs(ro[k])), (k, rg[k], ro[k])
    assert rg["balance_rel_max"] <= 1e-13 and rg["scale_rel_max"] <= 1e-13 and rg["neg_max"] == 0.0
    assert rg["newton_failures"] == 0


def test_checkpoint_resume():
    from paper_2602_22421_b200 import Solver
    inst = generate("small", m=400, N=200, k=(5, 60))
    a = Solver(inst, _params())
    a.step(20)
    y, y0 = a.primal()
    eta, s = a.duals(), a.usage()
    b = Solver(inst, _params())
    b.set_state(y=y, y0=y0, eta=eta, s_prev=s)
    a.step(10)
    b.step(10)
    ya, _ = a.primal()
    yb, _ = b.primal()
    assert rel_inf(yb, ya, 1.0) <= 1e-12 and rel_inf(b.duals(), a.duals(), 1.0) <= 1e-12
    a.close()
    b.close()


@pytest.mark.parametrize("sampled", [False, True])
def test_set_state_without_usage_recomputes_it(sampled):
    """spfom_set_state(y, y0, eta) without s_prev: the library recomputes
    s_prev = A y, so the resumed run equals the uninterrupted one (sampled
    mode: s_prev is the running stale-inclusive usage the next dual step adds
    its delta to)."""
    from paper_2602_22421_b200 import Solver
    inst = generate("small", m=400, N=200, k=(5, 60))
    blocks = block_sequence(inst.m, 90, 40, seed=4) if sampled else None
    p = _params(blocks=blocks, exec_mode=1)
    a = Solver(inst, p)
    a.step(20)
    y, y0 = a.primal()
    eta = a.duals()
    b = Solver(inst, p)
    b.step(20)                      # same block cursor; state then overwritten
    b.set_state(y=np.zeros_like(y), y0=inst.arrival.copy(), eta=np.zeros_like(eta))
    b.set_state(y=y, y0=y0, eta=eta)
    assert rel_inf(b.usage(), a.usage(), 1.0) <= 1e-12
    a.step(10)
    b.step(10)
    ya, _ = a.primal()
    yb, _ = b.primal()
    assert rel_inf(yb, ya, 1.0) <= 1e-12 and rel_inf(b.duals(), a.duals(), 1.0) <= 1e-12
    a.close()
    b.close()


def test_shadow_none_is_mnl():
    """shadow = NULL in the C ABI means MNL (w = 0): identical to explicit zeros."""
    import copy
    from paper_2602_22421_b200 import Solver
    inst = generate("small", m=300, N=150, k=(5, 40))
    inst.shadow[:] = 0.0
    inst2 = copy.copy(inst)
    inst2.shadow = None
    a, b = Solver(inst, _params()), Solver(inst2, _params())
    a.step(15)
    b.step(15)
    # equal up to the order of K1's fp64 global reductions (not fixed run to run)
    assert rel_inf(b.duals(), a.duals(), 1.0) <= 1e-12
    a.close()
    b.close()


def test_device_resident_instance():
    """spfom_instance.on_device = 1: torch CUDA tensors as the instance arrays
    give the same iterates as host arrays."""
    import copy
    import torch
    from paper_2602_22421_b200 import Solver
    inst = generate("medium", m=2000, N=1200, k=(20, 200))
    dev = copy.copy(inst)
    for f in ("seg_ptr", "prod_idx", "attract", "shadow", "no_purchase", "arrival", "price", "capacity"):
        setattr(dev, f, torch.from_numpy(np.ascontiguousarray(getattr(inst, f))).cuda())
    a, b = Solver(inst, _params()), Solver(dev, _params())
    a.step(10)
    b.step(10)
    ya, _ = a.primal()
    yb, _ = b.primal()
    assert rel_inf(yb, ya, 1.0) <= 1e-12 and rel_inf(b.duals(), a.duals(), 1.0) <= 1e-12
    a.close()
    b.close()


@pytest.mark.skipif("__import__('torch').cuda.device_count() < 2")
def test_two_devices_in_one_process():
    """Distinct handles on distinct GPUs are independent (per-device kernel
    attributes; every entry point runs on its handle's device)."""
    import torch
    from paper_2602_22421_b200 import Solver
    inst = generate("medium", m=3000, N=1500, k=(20, 200))
    a = Solver(inst, _params(), device="cuda:0")
    b = Solver(inst, _params(), device="cuda:1")
    torch.cuda.set_device(0)
    a.step(5)
    b.step(5)
    assert rel_inf(b.duals(), a.duals(), 1.0) <= 1e-12
    a.close()
    b.close()


def test_step_timed_is_step():
    """The timed stepping bench.py uses (two graphs per iteration, events around
    the primal graph) computes the same iterates as spfom_step."""
    from paper_2602_22421_b200 import Solver
    inst = generate("medium", m=3000, N=2000, k=(20, 200))
    a, b = Solver(inst, _params()), Solver(inst, _params())
    a.step(12)
    primal_ms, total_ms = b.step_timed(12)
    assert b.iteration == a.iteration == 12 and 0.0 < primal_ms <= total_ms
    ya, y0a = a.primal()
    yb, y0b = b.primal()
    assert rel_inf(yb, ya, 1.0) <= 1e-12 and rel_inf(y0b, y0a, 1.0) <= 1e-12
    assert rel_inf(b.duals(), a.duals(), 1.0) <= 1e-12
    a.close()
    b.close()


def test_pinned_pool_reuse_across_handles():
    """The pinned staging ring comes from a process-wide pool (spfom_create):
    handles alive together hold distinct buffers, a destroyed handle's buffers
    serve the next one, and create's layout and the getters' D2H through reused
    buffers give the same iterates (multi-chunk instance: > 2^18 quads), up to
    the rounding order of the usage reductions."""
    import threading
    from paper_2602_22421_b200 import Solver
    inst = generate("medium", m=12000, N=3000, k=(20, 200))    # ~1.3 M entries: several ring chunks
    ref = Solver(inst, _params())
    ref.step(6)
    y_ref, y0_ref = ref.primal()
    eta_ref = ref.duals()
    ref.close()                                                # its buffers go back to the pool
    out = {}

    def run(key):
        s = Solver(inst, _params())
        s.step(6)
        out[key] = (s.primal(), s.duals())
        s.close()
    threads = [threading.Thread(target=run, args=(k,)) for k in range(3)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert sorted(out) == [0, 1, 2]
    # equal up to the rounding order of the usage reductions (fp64 atomics):
    # a buffer shared by two live handles would differ at O(1)
    for (y, y0), eta in out.values():
        assert rel_inf(y, y_ref, 1.0) <= 1e-12 and rel_inf(y0, y0_ref, 1.0) <= 1e-12
        assert rel_inf(eta, eta_ref, 1.0) <= 1e-12


# ------------------------------------------------------------ accuracy gates
@pytest.mark.parametrize("seed", [1, 11, 12])
def test_tiny_accuracy_vs_dense_lp(seed):
    from paper_2602_22421_b200 import Solver
    inst = generate("tiny", seed=seed)
    Pstar = lp.sblp_dense(inst)[0]
    gpu = Solver(inst, _params())
    gpu.step(2000)
    r = gpu.residuals()
    gpu.close()
    assert abs(r["primal_obj"] - Pstar) <= 1e-6 * Pstar and r["infeas_rel"] <= 1e-6


def test_small_accuracy_vs_highs():
    from paper_2602_22421_b200 import Solver
    gold = json.load(open(GOLD))["small"]
    inst = generate("small")
    gpu = Solver(inst, _params())
    gpu.step(3000)
    r = gpu.residuals()
    gpu.close()
    assert abs(r["primal_obj"] - gold["Pstar"]) <= 1e-6 * gold["Pstar"], (r, gold)
    assert r["infeas_rel"] <= 1e-6
    assert r["cert_lower"] <= gold["Pstar"] * (1 + 1e-9) and gold["Pstar"] <= r["cert_upper"] * (1 + 1e-9)


# ------------------------------------------------------------ full-size sampled checks
def _check_sampled_segments(inst, gpu, eta_prev, y_prev, y0_prev, n_sample=3000, seed=0):
    """After one iteration from (y_prev, y0_prev, eta_prev), every segment's new
    row is the oracle projection of its own gradient step -- computable one by one."""
    rng = np.random.default_rng(seed)
    y, y0 = gpu.primal()
    g = inst.price - eta_prev
    worst = 0.0
    for i in rng.choice(inst.m, size=min(n_sample, inst.m), replace=False):
        sl = inst.row(int(i))
        z = y_prev[sl] + 1.0 * g[inst.prod_idx[sl]]
        r0, ry, _m, _ = oracle.project(y0_prev[i], z, inst.attract[sl], inst.shadow[sl], inst.no_purchase[i],
                                       inst.arrival[i])
        lam = inst.arrival[i]
        worst = max(worst, abs(y0[i] - r0) / lam, float(np.abs(y[sl] - ry).max()) / lam if ry.size else 0.0)
    return worst, y, y0


def test_multi_period_shared_structure_equals_stacked():
    """The shared-structure layout (num_periods = T, K1 k_primal_mp) and the
    same instance passed stacked as one period (K1 k_primal_stream) compute the
    same iterates; lengths cross the (4,4), (16,2) and (32,2) bins."""
    from paper_2602_22421_b200 import Solver
    inst = generate("multi", m=1500, N=900, k=(20, 200), T=4)
    a = Solver(inst, _params())
    b = Solver(inst, _params(), shared_periods=False)
    assert a.info()["num_periods"] == 4 and b.info()["num_periods"] == 1
    a.step(30)
    b.step(30)
    ya, y0a = a.primal()
    yb, y0b = b.primal()
    lam = float(inst.arrival.max())
    assert rel_inf(ya, yb, lam) <= 1e-12 and rel_inf(y0a, y0b, lam) <= 1e-12
    assert rel_inf(a.duals(), b.duals(), float(inst.price.max())) <= 1e-12
    ra, rb = a.residuals(), b.residuals()
    assert abs(ra["primal_obj"] - rb["primal_obj"]) <= 1e-12 * abs(rb["primal_obj"])
    assert abs(ra["dual_obj"] - rb["dual_obj"]) <= 1e-12 * abs(rb["dual_obj"])
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["medium", "huge", "multi"])
def test_full_size_sampled_outputs(name):
    """BASELINE full sizes in the bench launch configuration: sampled segment
    rows vs the oracle's projection, the usage vector vs a fresh sum, and eta
    vs the oracle's Eq. 17 step on that usage."""
    from paper_2602_22421_b200 import Solver
    inst = generate(name)
    gpu = Solver(inst, _params())
    gpu.step(3)
    y_prev, y0_prev = gpu.primal()
    eta_prev, s_prev = gpu.duals(), gpu.usage()
    gpu.step(1)
    worst, y, y0 = _check_sampled_segments(inst, gpu, eta_prev, y_prev, y0_prev)
    assert worst <= 1e-12, worst
    s = gpu.usage()
    fresh = np.bincount(inst.prod_idx, weights=y, minlength=inst.N)
    assert rel_inf(s, fresh, 1.0) <= 1e-12
    cpu = oracle.OracleSolver(generate("tiny"))       # only for tau_j via the oracle's own rule
    n = np.bincount(inst.prod_idx, minlength=inst.N)
    tau_j = np.where(n > 0, 0.9 / np.maximum(n, 1), 0.9)
    eta_ref = oracle.dual_step(eta_prev, s, s_prev, inst.capacity, tau_j, 0.0, 1.0)
    assert rel_inf(gpu.duals(), eta_ref, float(inst.price.max())) <= 1e-12
    r = gpu.residuals()
    gpu.close()
    assert r["newton_failures"] == 0 and r["balance_rel_max"] <= 1e-12 and r["neg_max"] == 0.0
    del cpu


def test_newton_budget_exhaustion_is_reported():
    """Failure detection: with a 2-pass budget the projection cannot finish; the
    next synchronising getter reports SPFOM_ENUMERIC and residuals count it."""
    from paper_2602_22421_b200 import Solver, SpfomError
    inst = generate("small", m=300, N=150, k=(5, 40))
    gpu = Solver(inst, _params(max_newton=2))
    gpu.step(3)
    r = gpu.residuals()
    assert r["newton_failures"] > 0
    with pytest.raises(SpfomError) as ei:
        gpu.duals()
    assert ei.value.status == 3
    gpu.close()


# ------------------------------------------------------------ SBLP -> CBLP recovery
def _check_recovery(inst, gpu, rows, exact_oracle=True):
    """GPU recovery vs the oracle's, computed from the GPU's own iterate (same
    u = y / v, so the order -- ties by product id -- is unique and must match
    exactly; alpha within 1e-12), plus the policy reproducing the row."""
    y, y0 = gpu.primal()
    order, alpha = gpu.recover()
    worst = 0.0
    for i in rows:
        sl = inst.row(int(i))
        k = sl.stop - sl.start
        o_pos, a_ref = oracle.recover(y0[i], y[sl], inst.attract[sl], inst.shadow[sl], inst.no_purchase[i],
                                      inst.arrival[i], inst.prod_idx[sl])
        got_o = order[sl]
        got_a = alpha[sl.start + i: sl.stop + i + 1]
        assert np.array_equal(got_o, inst.prod_idx[sl][o_pos]), (i, got_o, inst.prod_idx[sl][o_pos])
        worst = max(worst, float(np.abs(got_a - a_ref).max()))
        assert abs(got_a.sum() - 1.0) <= 1e-10 and got_a.min() >= -1e-12
        pos = {int(p): q for q, p in enumerate(inst.prod_idx[sl])}
        q0, q = oracle.policy_probabilities([pos[int(p)] for p in got_o], got_a, inst.attract[sl], inst.shadow[sl],
                                            inst.no_purchase[i])
        lam = inst.arrival[i]
        assert np.abs(lam * q - y[sl]).max() <= 1e-10 * lam and abs(lam * q0 - y0[i]) <= 1e-10 * lam
        del k
    return worst


@pytest.mark.parametrize("name,kw,iters", [("small", {}, 300), ("medium", dict(m=1500, N=1200, k=(20, 200)), 200),
                                           ("tiny", {}, 50)])
def test_recover_matches_oracle(name, kw, iters):
    from paper_2602_22421_b200 import Solver
    inst = generate(name, **kw)
    gpu = Solver(inst, _params())
    gpu.step(iters)
    worst = _check_recovery(inst, gpu, range(inst.m))
    # the timing helper runs the same launches into the workspace only: the
    # host-visible results of a later recover() are unchanged
    order, alpha = gpu.recover()
    assert gpu.recover_timed() > 0.0
    order2, alpha2 = gpu.recover()
    assert np.array_equal(order, order2) and np.array_equal(alpha, alpha2)
    gpu.close()
    assert worst <= 1e-12, worst


def test_recover_multi_period_and_full_size():
    from paper_2602_22421_b200 import Solver
    inst = generate("multi", m=600, N=500, k=(10, 120), T=3)
    gpu = Solver(inst, _params())
    gpu.step(60)
    assert _check_recovery(inst, gpu, range(0, inst.m, 7)) <= 1e-12
    gpu.close()
    inst = generate("huge")
    gpu = Solver(inst, _params())
    gpu.step(5)
    rows = np.random.default_rng(3).choice(inst.m, 300, replace=False)
    assert _check_recovery(inst, gpu, rows) <= 1e-12
    gpu.close()


# ------------------------------------------------------------ bundles / NRM (Eq. 33)
@pytest.mark.parametrize("name,kw,L,blocks_B", [
    ("small", dict(m=400, N=120, k=(5, 40)), 40, None),
    ("medium", dict(m=2000, N=1500, k=(20, 200)), 500, None),        # several bins, Zipf head
    ("small", dict(m=600, N=200, k=(5, 40)), 64, 150),               # sampled blocks
    ("multi", dict(m=300, N=200, k=(5, 60), T=3), 70, None),         # shared periods
])
def test_bundle_lockstep_100(name, kw, L, blocks_B):
    from spfom_inputs import with_bundles
    inst = with_bundles(generate(name, **kw), L=L, seed=2)
    blocks = None if blocks_B is None else block_sequence(inst.m, blocks_B, 32, 5)
    worst, gpu, cpu = lockstep(inst, _params(blocks=blocks), 100, blocks=blocks)
    assert gpu.duals().shape == (L,)
    rg, ro = gpu.residuals(), cpu.residuals()
    gpu.close()
    _assert_ok(worst)
    for k in ("primal_obj", "dual_obj", "cert_lower", "cert_upper"):
        assert abs(rg[k] - ro[k]) <= 1e-10 * abs(ro[k]), (k, rg[k], ro[k])
    for k in ("infeas_abs", "infeas_rel", "alpha", "compl_slack"):
        assert abs(rg[k] - ro[k]) <= 1e-10 * max(1.0, abs(ro[k])), (k, rg[k], ro[k])


def test_bundle_identity_incidence_equals_plain_path():
    """Reduction law on the GPU: Bt = I runs the bundle dual kernels
    yet reproduces the per-product path."""
    from paper_2602_22421_b200 import Solver
    from spfom_inputs import with_bundles
    inst = generate("medium", m=1500, N=900, k=(20, 120))
    a, b = Solver(inst, _params(exec_mode=1)), Solver(with_bundles(inst, identity=True), _params())
    a.step(40)
    b.step(40)
    ya, _ = a.primal()
    yb, _ = b.primal()
    assert rel_inf(yb, ya, 1.0) <= 1e-12 and rel_inf(b.duals(), a.duals(), 1.0) <= 1e-12
    a.close()
    b.close()


# ------------------------------------------------------------ feature combinations
@pytest.mark.parametrize("combo", ["paper-multi", "paper-bundles", "averaging-bundles", "averaging-multi",
                                   "ragged-graph", "paper-medium-graph"])
def test_feature_combinations_lockstep(combo):
    """The layouts x presets the kernels branch on: exact argmax through the
    shared-period kernel and with bundle prices, averaging with resource duals
    and with [T][m] segment state, the ragged-bin instance and the paper preset
    through the per-iteration graph instead of the persistent small kernel."""
    from paper_2602_22421_b200 import Params
    from spfom_inputs import with_bundles
    if combo == "paper-multi":
        inst, p, iters = generate("multi", m=300, N=200, k=(5, 60), T=3), Params.paper(mu=0.3), 60
    elif combo == "paper-bundles":
        inst = with_bundles(generate("small", m=400, N=150, k=(5, 40)), L=50, seed=6)
        p, iters = Params.paper(mu=0.3), 60
    elif combo == "averaging-bundles":
        inst = with_bundles(generate("small", m=400, N=150, k=(5, 40)), L=50, seed=7)
        p, iters = _params(averaging=True), 40
    elif combo == "averaging-multi":
        inst, p, iters = generate("multi", m=300, N=200, k=(5, 60), T=2), _params(averaging=True), 40
    elif combo == "ragged-graph":
        ks = [0, 1, 3, 16, 17, 33, 64, 65, 129, 257, 513, 1000, 50] * 4
        inst, p, iters = _ragged_instance(ks, N=1100, seed=2), _params(exec_mode=1), 40
    else:
        inst, p, iters = generate("medium", m=1500, N=1000, k=(20, 200)), Params.paper(mu=0.0, exec_mode=1), 60
    worst, gpu, cpu = lockstep(inst, p, iters)
    if p.averaging:
        yb, y0b, eb = gpu.averages()
        lam, rmax = float(inst.arrival.max()), float(inst.price.max())
        assert rel_inf(yb, cpu.ybar, lam) <= TOL_ITER and rel_inf(y0b, cpu.y0bar, lam) <= TOL_ITER
        assert rel_inf(eb, cpu.etabar, rmax) <= TOL_ITER
    gpu.close()
    _assert_ok(worst)


@pytest.mark.parametrize("collective", ["reduce_scatter", "allreduce"])
@pytest.mark.parametrize("name,kw", [("medium", dict(m=30000, N=4000, k=(20, 200))),
                                     ("multi", dict(m=3000, N=800, k=50, T=3))])
def test_nccl_path_single_rank(name, kw, collective, monkeypatch):
    """The multi-rank code path (ncclCommInitRank from a unique id, k_fold of the
    spread copies, global column counts by allreduce, and per iteration either
    ReduceScatter -> K3 on the rank's slice -> AllGather of the prices (the
    default for world > 1) or an allreduce + replicated K3
    (SPFOM_COLLECTIVE=allreduce), inside the CUDA graph), run with world == 1
    on this GPU for 100 iterations: iterates equal to the single-GPU path up
    to the order of the fp64 reductions (K1's global RED order is not fixed, so
    two runs are not bitwise equal) and within 1e-10 of the oracle every 10
    iterations; the getters gather the sliced duals / usage."""
    from paper_2602_22421_b200 import Params, Solver, nccl_unique_id
    if collective == "allreduce":
        monkeypatch.setenv("SPFOM_COLLECTIVE", "allreduce")
    inst = generate(name, **kw)
    p = Params.converge(exec_mode=1)
    a = Solver(inst, p)
    b = Solver(inst, p, rank=0, world=1, nccl_id=nccl_unique_id())
    assert b.info()["launches_per_iteration"] == a.info()["launches_per_iteration"] + 1   # + k_fold
    cpu = oracle.OracleSolver(inst, **oracle_kwargs(p))
    lam, rmax = float(inst.arrival.max()), float(inst.price.max())
    for t in range(100):
        a.step(1)
        b.step(1)
        cpu.step()
        if (t + 1) % 10 == 0:
            yb, y0b = b.primal()
            assert rel_inf(yb, cpu.y, lam) <= TOL_ITER and rel_inf(b.duals(), cpu.eta, rmax) <= TOL_ITER, t
            assert rel_inf(b.usage(), cpu.s, lam) <= TOL_ITER
    ya, y0a = a.primal()
    yb, y0b = b.primal()
    assert rel_inf(yb, ya, lam) <= 1e-12 and rel_inf(y0b, y0a, lam) <= 1e-12
    assert rel_inf(b.duals(), a.duals(), rmax) <= 1e-12
    ra, rb = a.residuals(), b.residuals()
    assert abs(ra["primal_obj"] - rb["primal_obj"]) <= 1e-12 * abs(ra["primal_obj"])
    assert abs(ra["dual_obj"] - rb["dual_obj"]) <= 1e-12 * abs(ra["dual_obj"])
    a.close()
    b.close()
