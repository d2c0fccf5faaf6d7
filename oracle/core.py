"""ctypes wrapper of oracle/spfom_oracle.c (test infrastructure only)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spfom_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

residual_names = ("primal_obj", "dual_obj", "rel_gap", "infeas_abs", "infeas_rel", "infeas_rel_l2",
                  "balance_rel_max", "scale_rel_max", "neg_max", "compl_slack", "cert_lower",
                  "cert_upper", "alpha")


def build_oracle(force: bool = False) -> str:
    """gcc -O2 -ffp-contract=off (reading c14: no FMA contraction in the oracle)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
                               "-Wall", "-shared", "-fPIC", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class _Inst(C.Structure):
    _fields_ = [("m", C.c_int64), ("N", C.c_int64), ("seg_ptr", C.c_void_p), ("prod_idx", C.c_void_p),
                ("v", C.c_void_p), ("w", C.c_void_p), ("v0", C.c_void_p), ("lam", C.c_void_p),
                ("r", C.c_void_p), ("c", C.c_void_p), ("L", C.c_int64), ("bptr", C.c_void_p),
                ("bres", C.c_void_p), ("cres", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("theta", C.c_double), ("mu", C.c_double), ("extrapolation", C.c_double),
                ("averaging", C.c_int32), ("pad_", C.c_int32), ("refresh_every", C.c_int64)]


class _State(C.Structure):
    _fields_ = [("y", C.c_void_p), ("y0", C.c_void_p), ("eta", C.c_void_p), ("s", C.c_void_p),
                ("ybar", C.c_void_p), ("y0bar", C.c_void_p), ("etabar", C.c_void_p), ("t", C.c_int64)]


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build_oracle())
        L.oracle_project.restype = C.c_int
        L.oracle_project.argtypes = [C.c_int64, C.c_double, _dp, _dp, _dp, C.c_double, C.c_double,
                                     C.POINTER(C.c_double), _dp, _dp, C.POINTER(C.c_int)]
        L.oracle_argmax.restype = C.c_double
        L.oracle_argmax.argtypes = [C.c_int64, _dp, _dp, _dp, C.c_double, C.c_double,
                                    C.POINTER(C.c_double), _dp, C.POINTER(C.c_double)]
        L.oracle_fast_inner.restype = C.c_double
        L.oracle_fast_inner.argtypes = [C.c_int64, _dp, _dp, C.c_double, C.c_double, C.c_double, _dp]
        L.oracle_golden.restype = C.c_double
        L.oracle_golden.argtypes = [C.c_int64, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_double), _dp]
        L.oracle_dual_step.restype = None
        L.oracle_dual_step.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double]
        L.oracle_tau.restype = None
        L.oracle_tau.argtypes = [C.POINTER(_Inst), C.c_double, C.c_int, _dp]
        L.oracle_init.restype = None
        L.oracle_init.argtypes = [C.POINTER(_Inst), C.POINTER(_State)]
        L.oracle_iterate.restype = C.c_int
        L.oracle_iterate.argtypes = [C.POINTER(_Inst), C.POINTER(_Params), _dp, C.c_void_p, C.c_int64,
                                     C.POINTER(_State)]
        L.oracle_primal_shard.restype = C.c_int
        L.oracle_primal_shard.argtypes = [C.POINTER(_Inst), C.POINTER(_Params), C.POINTER(_State), _dp]
        L.oracle_dual_apply.restype = None
        L.oracle_dual_apply.argtypes = [C.POINTER(_Inst), C.POINTER(_Params), _dp, _dp, C.POINTER(_State)]
        L.oracle_recover.restype = None
        L.oracle_recover.argtypes = [C.c_int64, C.c_double, _dp, _dp, _dp, C.c_double, C.c_double, _ip, _lp, _dp]
        L.oracle_prices.restype = None
        L.oracle_prices.argtypes = [C.POINTER(_Inst), _dp, _dp]
        L.oracle_residuals.restype = C.c_int
        L.oracle_residuals.argtypes = [C.POINTER(_Inst), _dp, _dp, _dp, C.c_void_p, _dp]
        _lib = L
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def recover(y0, y, v, w, v0, lam, prod):
    """SBLP -> CBLP recovery of one row (GAM reading): returns
    (order, alpha) -- row positions of the products by y/v descending (ties:
    ascending product id) and the probabilities alpha(S_0..S_k) of the nested
    assortments S_l = first l products (S_0: no-purchase only)."""
    y, v, w = _f64(y), _f64(v), _f64(w)
    prod = np.ascontiguousarray(prod, dtype=np.int32)
    k = y.shape[0]
    order = np.zeros(k, dtype=np.int64)
    alpha = np.zeros(k + 1)
    lib().oracle_recover(k, float(y0), y, v, w, float(v0), float(lam), prod, order, alpha)
    return order, alpha


def policy_probabilities(order, alpha, v, w, v0):
    """Per-entry sales share of a recovered policy under GAM choice:
    returns (q0, q) with q_j = sum_l alpha_l pi_j(S_l), q0 = sum_l alpha_l pi_0(S_l),
    pi_j(S) = v_j / D(S) on S, pi_0(S) = (v0 + sum_{C \\ S} w) / D(S).  Plain
    definition, used to check the recovery against the row it came from."""
    v, w = _f64(v), _f64(w)
    k = v.shape[0]
    q = np.zeros(k)
    q0 = 0.0
    for l in range(k + 1):
        S = set(int(x) for x in order[:l])
        D = v0 + sum(v[j] if j in S else w[j] for j in range(k))
        for j in S:
            q[j] += alpha[l] * v[j] / D
        q0 += alpha[l] * (v0 + sum(w[j] for j in range(k) if j not in S)) / D
    return q0, q


def project(z0, z, v, w, v0, lam):
    """Pi_{Y_i}(z0, z) -> (y0, y, (nu, kappa, U), evaluations).  Raises on failure."""
    z, v, w = _f64(z), _f64(v), _f64(w)
    y = np.zeros(z.shape[0])
    mult = np.zeros(3)
    y0 = C.c_double()
    it = C.c_int()
    rc = lib().oracle_project(z.shape[0], float(z0), z, v, w, float(v0), float(lam), C.byref(y0), y, mult,
                              C.byref(it))
    if rc != 0:
        raise FloatingPointError(f"oracle_project failed (status {rc})")
    return y0.value, y, mult, it.value


def argmax(g, v, w, v0, lam):
    """Exact inner argmax -> (value lambda*z*, y0, y, tie margin)."""
    g, v, w = _f64(g), _f64(v), _f64(w)
    y = np.zeros(g.shape[0])
    y0 = C.c_double()
    mg = C.c_double()
    val = lib().oracle_argmax(g.shape[0], g, v, w, float(v0), float(lam), C.byref(y0), y, C.byref(mg))
    return val, y0.value, y, mg.value


def fast_inner(g, v, v0, lam, y0):
    """Algorithm 1 (MNL) for fixed y0 -> (z_i, y); z_i is NaN below the feasibility bound."""
    g, v = _f64(g), _f64(v)
    y = np.zeros(g.shape[0])
    val = lib().oracle_fast_inner(g.shape[0], g, v, float(v0), float(lam), float(y0), y)
    return val, y


def golden(g, v, v0, lam, tol=1e-3):
    """Golden-section search over y0 with FAST-INNER -> (value, y0, y)."""
    g, v = _f64(g), _f64(v)
    y = np.zeros(g.shape[0])
    y0 = C.c_double()
    val = lib().oracle_golden(g.shape[0], g, v, float(v0), float(lam), float(tol), C.byref(y0), y)
    return val, y0.value, y


def dual_step(eta, s_new, s_old, c, tau_j, mu=0.0, omega_x=0.0):
    """Eq. 17 on the extrapolated usage -> new eta (array)."""
    eta = _f64(eta).copy()
    lib().oracle_dual_step(eta.shape[0], eta, _f64(s_new), _f64(s_old), _f64(c), _f64(tau_j),
                           float(mu), float(omega_x))
    return eta


def compute_R(inst) -> float:
    """R = max_i sum_j v_ij r_j / sum_j v_ij (Theorem 2)."""
    best = -np.inf
    for i in range(inst.m):
        sl = inst.row(i)
        v = inst.attract[sl]
        best = max(best, float((v * inst.price[inst.prod_idx[sl]]).sum() / v.sum()))
    return best


class OracleSolver:
    """Single-threaded SPFOM on the CPU, one `step()` = one iteration.

    Parameters follow SURVEY §8(b)/(c): theta (inf => exact argmax), tau with
    tau_mode 0 (scalar) / 1 (tau / n_j), mu (Eq. 17), extrapolation omega_x,
    averaging, refresh_every (sampled mode)."""

    def __init__(self, inst, theta=1.0, tau=0.9, tau_mode=1, mu=0.0, extrapolation=1.0,
                 averaging=False, refresh_every=0):
        self.inst = inst
        self._keep = dict(
            seg_ptr=np.ascontiguousarray(inst.seg_ptr, dtype=np.int64),
            prod_idx=np.ascontiguousarray(inst.prod_idx, dtype=np.int32),
            v=_f64(inst.attract), w=_f64(inst.shadow), v0=_f64(inst.no_purchase),
            lam=_f64(inst.arrival), r=_f64(inst.price), c=_f64(inst.capacity))
        k = self._keep
        # bundles (NRM): resources of bundle j = bundle_res[bundle_ptr[j]:bundle_ptr[j+1]]
        L = int(getattr(inst, "num_resources", 0) or 0)
        if L > 0:
            k.update(bptr=np.ascontiguousarray(inst.bundle_ptr, dtype=np.int64),
                     bres=np.ascontiguousarray(inst.bundle_res, dtype=np.int32),
                     cres=_f64(inst.resource_capacity))
        self.L = L
        self._inst = _Inst(inst.m, inst.N, *[k[n].ctypes.data for n in
                                             ("seg_ptr", "prod_idx", "v", "w", "v0", "lam", "r", "c")],
                           L, *([k[n].ctypes.data for n in ("bptr", "bres", "cres")] if L > 0 else [None] * 3))
        nd = L if L > 0 else inst.N              # duals: per resource (bundles) or per product
        self._params = _Params(float(theta), float(mu), float(extrapolation), int(bool(averaging)), 0,
                               int(refresh_every))
        self.tau_j = np.zeros(nd)
        lib().oracle_tau(C.byref(self._inst), float(tau), int(tau_mode), self.tau_j)
        self.y = np.zeros(inst.nnz)
        self.y0 = np.zeros(inst.m)
        self.eta = np.zeros(nd)
        self.s = np.zeros(inst.N)
        self.averaging = bool(averaging)
        if self.averaging:
            self.ybar = np.zeros(inst.nnz)
            self.y0bar = np.zeros(inst.m)
            self.etabar = np.zeros(nd)
        self._state = _State(self.y.ctypes.data, self.y0.ctypes.data, self.eta.ctypes.data,
                             self.s.ctypes.data,
                             self.ybar.ctypes.data if self.averaging else None,
                             self.y0bar.ctypes.data if self.averaging else None,
                             self.etabar.ctypes.data if self.averaging else None, 0)
        lib().oracle_init(C.byref(self._inst), C.byref(self._state))

    @property
    def t(self) -> int:
        return int(self._state.t)

    def step(self, block: Optional[np.ndarray] = None) -> None:
        if block is None:
            rc = lib().oracle_iterate(C.byref(self._inst), C.byref(self._params), self.tau_j, None,
                                      self.inst.m, C.byref(self._state))
        else:
            blk = np.ascontiguousarray(block, dtype=np.int32)
            rc = lib().oracle_iterate(C.byref(self._inst), C.byref(self._params), self.tau_j,
                                      blk.ctypes.data, blk.shape[0], C.byref(self._state))
        if rc != 0:
            raise FloatingPointError(f"oracle_iterate failed at t={self.t} (status {rc})")

    # --- sharded emulation (Alg. 3): the caller sums the ranks' usage ---------
    def primal_shard(self) -> np.ndarray:
        """Full-sweep primal step of this (shard) instance; returns its usage."""
        s_local = np.zeros(self.inst.N)
        rc = lib().oracle_primal_shard(C.byref(self._inst), C.byref(self._params), C.byref(self._state), s_local)
        if rc != 0:
            raise FloatingPointError(f"oracle_primal_shard failed (status {rc})")
        return s_local

    def dual_apply(self, s_global: np.ndarray) -> None:
        """Dual step with the global usage (identical on every rank)."""
        lib().oracle_dual_apply(C.byref(self._inst), C.byref(self._params), self.tau_j, _f64(s_global),
                                C.byref(self._state))

    def run(self, iters: int, blocks: Optional[np.ndarray] = None) -> None:
        for t in range(iters):
            self.step(None if blocks is None else blocks[self.t % blocks.shape[0]])

    def prices(self, eta=None) -> np.ndarray:
        """g = r - A^T eta (bundles: r_j - sum_{l in B_j} eta_l)."""
        g = np.zeros(self.inst.N)
        lib().oracle_prices(C.byref(self._inst), _f64(self.eta if eta is None else eta), g)
        return g

    def residuals(self, eta=None, y=None, y0=None) -> dict:
        out = np.zeros(len(residual_names))
        present = np.ascontiguousarray(self.inst.present, dtype=np.uint8)
        lib().oracle_residuals(C.byref(self._inst), _f64(self.eta if eta is None else eta),
                               _f64(self.y if y is None else y), _f64(self.y0 if y0 is None else y0),
                               present.ctypes.data, out)
        return dict(zip(residual_names, out.tolist()))
