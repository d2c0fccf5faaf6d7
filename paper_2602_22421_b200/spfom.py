"""Thin ctypes binding of include/spfom.h (argument marshalling only).

Every step of the SPFOM iteration runs in libspfom.so's CUDA kernels; this
module only converts numpy arrays to pointers, allocates the device workspace
with PyTorch (device memory + streams are PyTorch's job here) and exposes the
same names as the C ABI.  There is no CPU fallback: if the library or a CUDA
device is missing the calls raise.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPFOM_LIB") or os.path.join(_HERE, "libspfom.so")

STATUS = {0: "SPFOM_OK", 1: "SPFOM_EINVAL", 2: "SPFOM_EDATA", 3: "SPFOM_ENUMERIC", 4: "SPFOM_ECUDA",
          5: "SPFOM_ENCCL", 6: "SPFOM_ENOMEM"}

EXPORTED = ("spfom_workspace_bytes", "spfom_create", "spfom_step", "spfom_duals", "spfom_primal", "spfom_usage",
            "spfom_averages", "spfom_objective", "spfom_residuals", "spfom_set_state", "spfom_info",
            "spfom_time_kernels", "spfom_step_timed", "spfom_recover", "spfom_recover_timed", "spfom_iteration",
            "spfom_last_error", "spfom_destroy", "spfom_partition", "spfom_nccl_unique_id", "spfom_build_info",
            "spfom_abi_sizes")


class SpfomError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Instance(C.Structure):
    _fields_ = [("num_segments", C.c_int64), ("num_products", C.c_int64), ("nnz", C.c_int64),
                ("segment_offset", C.c_int64), ("num_segments_global", C.c_int64),
                ("seg_ptr", C.c_void_p), ("prod_idx", C.c_void_p), ("attract", C.c_void_p),
                ("shadow", C.c_void_p), ("no_purchase", C.c_void_p), ("arrival", C.c_void_p),
                ("price", C.c_void_p), ("capacity", C.c_void_p), ("num_periods", C.c_int64),
                ("num_resources", C.c_int64), ("bundle_ptr", C.c_void_p), ("bundle_res", C.c_void_p),
                ("resource_capacity", C.c_void_p), ("on_device", C.c_int64)]


class _Params(C.Structure):
    _fields_ = [("theta", C.c_double), ("tau", C.c_double), ("mu", C.c_double), ("extrapolation", C.c_double),
                ("tau_mode", C.c_int32), ("averaging", C.c_int32), ("max_newton", C.c_int32),
                ("exec_mode", C.c_int32), ("block_size", C.c_int64), ("block_iters", C.c_int64),
                ("blocks", C.c_void_p), ("refresh_every", C.c_int64)]


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p)]


class _Residuals(C.Structure):
    _fields_ = [("iteration", C.c_int64)] + [(n, C.c_double) for n in (
        "primal_obj", "dual_obj", "rel_gap", "infeas_abs", "infeas_rel", "infeas_rel_l2", "balance_rel_max",
        "scale_rel_max", "neg_max", "compl_slack", "cert_lower", "cert_upper", "alpha")] + [
        ("newton_failures", C.c_int64), ("newton_passes", C.c_int64), ("newton_restarts", C.c_int64)]


class _Info(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("num_segments", "num_products", "nnz", "nnz_padded", "n_present",
                                          "launches_per_iteration", "primal_launches_per_iteration",
                                          "workspace_bytes")] + [
        ("bin_segments", C.c_int64 * 8), ("bin_G", C.c_int32 * 8), ("bin_Q", C.c_int32 * 8),
        ("num_bins", C.c_int32), ("world", C.c_int32), ("num_periods", C.c_int64), ("persistent", C.c_int64)]


_lib = None


def _base_of_stacked(inst, T: int) -> dict:
    """Base rows of a period-major stacked instance (segment t*m + i = base row i
    in period t; SPEC stack_periods), checked to really share the structure."""
    M = int(inst.seg_ptr.shape[0] - 1)
    if M % T:
        raise SpfomError(2, f"stacked instance has {M} segments, not a multiple of T = {T}")
    m = M // T
    nb = int(inst.seg_ptr[m])
    seg_ptr = np.asarray(inst.seg_ptr[: m + 1], dtype=np.int64)
    tiled = dict(prod_idx=nb, attract=nb, shadow=nb, no_purchase=m)
    for name, n in tiled.items():
        if getattr(inst, name, None) is None:
            continue
        a = np.asarray(getattr(inst, name))
        if a.shape[0] != n * T or not np.array_equal(a.reshape(T, n), np.broadcast_to(a[:n], (T, n))):
            raise SpfomError(2, f"multi-period instance: {name} differs across periods (no shared structure)")
    if not np.array_equal(np.asarray(inst.seg_ptr).reshape(-1)[1:].reshape(T, m) - np.arange(T)[:, None] * nb,
                          np.broadcast_to(seg_ptr[1:], (T, m))):
        raise SpfomError(2, "multi-period instance: consideration sets differ across periods")
    shadow = getattr(inst, "shadow", None)
    return dict(seg_ptr=seg_ptr, prod_idx=inst.prod_idx[:nb], attract=inst.attract[:nb],
                shadow=None if shadow is None else shadow[:nb],
                no_purchase=inst.no_purchase[:m], arrival=np.asarray(inst.arrival, dtype=np.float64))


def load_library() -> C.CDLL:
    """Load libspfom.so (in-tree).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i64, st = C.c_void_p, C.c_int64, C.c_int
        L.spfom_workspace_bytes.argtypes = [C.POINTER(_Instance), C.POINTER(_Params), C.POINTER(C.c_size_t)]
        L.spfom_create.argtypes = [C.POINTER(_Instance), C.POINTER(_Params), C.POINTER(_Dist), vp, vp, C.c_size_t,
                                   C.POINTER(vp)]
        L.spfom_step.argtypes = [vp, i64]
        L.spfom_duals.argtypes = [vp, vp]
        L.spfom_primal.argtypes = [vp, vp, vp]
        L.spfom_usage.argtypes = [vp, vp]
        L.spfom_averages.argtypes = [vp, vp, vp, vp]
        L.spfom_objective.argtypes = [vp, C.POINTER(C.c_double)]
        L.spfom_residuals.argtypes = [vp, C.POINTER(_Residuals)]
        L.spfom_set_state.argtypes = [vp, vp, vp, vp, vp]
        L.spfom_info.argtypes = [vp, C.POINTER(_Info)]
        L.spfom_time_kernels.argtypes = [vp, i64, vp]
        L.spfom_step_timed.argtypes = [vp, i64, vp]
        L.spfom_recover.argtypes = [vp, vp, vp]
        L.spfom_recover_timed.argtypes = [vp, vp]
        L.spfom_iteration.argtypes = [vp]
        L.spfom_iteration.restype = i64
        L.spfom_last_error.argtypes = [vp]
        L.spfom_last_error.restype = C.c_char_p
        L.spfom_destroy.argtypes = [vp]
        L.spfom_destroy.restype = None
        L.spfom_partition.argtypes = [vp, i64, C.c_int32, vp]
        L.spfom_nccl_unique_id.argtypes = [vp]
        L.spfom_build_info.restype = C.c_char_p
        for name in EXPORTED:
            if name not in ("spfom_iteration", "spfom_last_error", "spfom_destroy", "spfom_build_info"):
                getattr(L, name).restype = st
        _lib = L
    return _lib


def _check(status: int, handle=None):
    if status != 0:
        msg = load_library().spfom_last_error(handle)
        raise SpfomError(status, msg.decode() if msg else "")


@dataclasses.dataclass
class Params:
    """spfom_params; presets `paper()` and `converge()` (§8(c) c8)."""
    theta: float = 1.0
    tau: float = 0.9
    tau_mode: int = 1
    mu: float = 0.0
    extrapolation: float = 1.0
    averaging: bool = False
    blocks: Optional[np.ndarray] = None      # [iters][B] int32 global ids, rows sorted
    refresh_every: int = 0
    max_newton: int = 200
    exec_mode: int = 0                        # 0 auto, 1 graph per iteration, 2 persistent small regime

    @staticmethod
    def converge(**kw) -> "Params":
        return Params(**kw)

    @staticmethod
    def paper(mu: float = 0.0, tau: float = 0.1, blocks=None, **kw) -> "Params":
        return Params(theta=math.inf, tau=tau, tau_mode=0, mu=mu, extrapolation=0.0, blocks=blocks, **kw)

    def _c(self):
        blocks = None if self.blocks is None else np.ascontiguousarray(self.blocks, dtype=np.int32)
        p = _Params(float(self.theta), float(self.tau), float(self.mu), float(self.extrapolation), int(self.tau_mode),
                    int(bool(self.averaging)), int(self.max_newton), int(self.exec_mode),
                    0 if blocks is None else blocks.shape[1], 0 if blocks is None else blocks.shape[0],
                    None if blocks is None else blocks.ctypes.data, int(self.refresh_every))
        return p, blocks


def partition(seg_ptr: np.ndarray, world: int) -> np.ndarray:
    """spfom_partition: contiguous segment ranges balanced by nnz (host only)."""
    sp = np.ascontiguousarray(seg_ptr, dtype=np.int64)
    out = np.zeros(world + 1, dtype=np.int64)
    _check(load_library().spfom_partition(sp.ctypes.data, sp.shape[0] - 1, int(world), out.ctypes.data))
    return out


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(load_library().spfom_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _is_cuda_tensor(a) -> bool:
    return getattr(a, "is_cuda", False) is True


def _host_array(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _dev_array(a, dtype):
    import torch
    tdt = {np.int64: torch.int64, np.int32: torch.int32, np.float64: torch.float64}[dtype]
    return a.to(dtype=tdt).contiguous()


def _len(a) -> int:
    return int(a.shape[0])


def _ptr(a):
    if a is None:
        return None
    return a.data_ptr() if _is_cuda_tensor(a) else a.ctypes.data


class Solver:
    """One spfom handle.  `inst` is any object with the CSR fields of
    spfom_instance (seg_ptr, prod_idx, attract, shadow, no_purchase, arrival,
    price, capacity); with world > 1 it is this rank's shard and
    `segment_offset` / `num_segments_global` locate it."""

    def __init__(self, inst, params: Optional[Params] = None, *, device=None, stream=None,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 segment_offset: int = 0, num_segments_global: Optional[int] = None,
                 shared_periods: bool = True, workspace_offset_bytes: int = 0, workspace=None):
        """workspace: an optional caller-provided uint8 CUDA tensor of at least
        workspace_bytes(inst, params) + 256 bytes (spfom_create's workspace
        argument; the solver keeps a reference).
        workspace_offset_bytes > 0: a device allocation of that size is made
        (and kept for the solver's lifetime) before the workspace, which then
        lands above it -- a placement probe only: round 2 measured K1 the same
        at every offset from 0 to 96 GiB, and bench.py passes 0."""
        import torch  # device memory and streams only

        L = load_library()
        self.params = params or Params()
        arrays = dict(seg_ptr=inst.seg_ptr, prod_idx=inst.prod_idx, attract=inst.attract,
                      shadow=getattr(inst, "shadow", None), no_purchase=inst.no_purchase, arrival=inst.arrival)
        # a period-major stacked multi-period instance goes to the shared-structure
        # layout (num_periods = T): base rows once, arrival [T][m]
        T = int((getattr(inst, "meta", None) or {}).get("T", 1) or 1)
        self.periods = T if (shared_periods and T > 1) else 1
        # instance arrays already in device memory (torch CUDA tensors): passed as
        # device pointers (spfom_instance.on_device = 1), staged by the library
        on_dev = [_is_cuda_tensor(a) for a in list(arrays.values()) + [inst.price, inst.capacity] if a is not None]
        on_device = bool(on_dev) and all(on_dev)
        if any(on_dev) and not on_device:
            raise SpfomError(1, "instance arrays must be all host arrays or all CUDA tensors")
        if on_device and self.periods > 1:
            raise SpfomError(1, "device-resident instances: pass the base rows with num_periods (host layout check)")
        if self.periods > 1:
            arrays = _base_of_stacked(inst, T)
        conv = _dev_array if on_device else _host_array
        k = self._keep = dict(
            seg_ptr=conv(arrays["seg_ptr"], np.int64), prod_idx=conv(arrays["prod_idx"], np.int32),
            attract=conv(arrays["attract"], np.float64),
            shadow=None if arrays["shadow"] is None else conv(arrays["shadow"], np.float64),
            no_purchase=conv(arrays["no_purchase"], np.float64), arrival=conv(arrays["arrival"], np.float64),
            price=conv(inst.price, np.float64), capacity=conv(inst.capacity, np.float64))
        mb = _len(k["seg_ptr"]) - 1
        nb = _len(k["prod_idx"])
        self.m = mb * self.periods            # stacked sizes: the getters' shapes
        self.N = _len(k["price"])
        self.nnz = nb * self.periods
        # every length the library reads is checked here (it trusts the sizes)
        want = dict(attract=nb, shadow=nb, no_purchase=mb, arrival=self.periods * mb, capacity=self.N)
        for name, n in want.items():
            if k[name] is not None and _len(k[name]) != n:
                raise SpfomError(1, f"instance: len({name}) = {_len(k[name])}, expected {n}")
        if mb < 0 or self.N < 1:
            raise SpfomError(1, "instance: need seg_ptr of length m + 1 >= 1 and at least one product")
        # bundles / NRM: duals per resource
        self.L = int(getattr(inst, "num_resources", 0) or 0)
        if self.L > 0:
            k.update(bundle_ptr=conv(inst.bundle_ptr, np.int64), bundle_res=conv(inst.bundle_res, np.int32),
                     resource_capacity=conv(inst.resource_capacity, np.float64))
            if _len(k["bundle_ptr"]) != self.N + 1 or _len(k["resource_capacity"]) != self.L:
                raise SpfomError(1, "instance: bundle_ptr needs N + 1 entries and resource_capacity L")
        self.n_duals = self.L if self.L > 0 else self.N
        if not torch.cuda.is_available():
            raise SpfomError(4, "no CUDA device: the SPFOM path has no CPU fallback")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._inst = _Instance(mb, self.N, nb, int(segment_offset),
                               int(num_segments_global if num_segments_global is not None else mb),
                               *[_ptr(k[n]) for n in ("seg_ptr", "prod_idx", "attract", "shadow",
                                                      "no_purchase", "arrival", "price", "capacity")],
                               self.periods, self.L,
                               *([_ptr(k[n]) for n in ("bundle_ptr", "bundle_res", "resource_capacity")]
                                 if self.L > 0 else [None] * 3), int(on_device))
        self._params, self._blocks = self.params._c()
        nbytes = C.c_size_t()
        _check(L.spfom_workspace_bytes(C.byref(self._inst), C.byref(self._params), C.byref(nbytes)))
        with torch.cuda.device(self.device):
            # a dedicated stream: the legacy default stream cannot be captured into a CUDA graph
            self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
            self._placement_pad = (torch.empty(int(workspace_offset_bytes), dtype=torch.uint8, device=self.device)
                                   if workspace_offset_bytes > 0 else None)
            need = max(int(nbytes.value), 256) + 256
            if workspace is not None:
                if not _is_cuda_tensor(workspace) or workspace.dtype != torch.uint8 or workspace.numel() < need:
                    raise SpfomError(6, f"workspace: need a uint8 CUDA tensor of >= {need} bytes")
                self.workspace = workspace
            else:
                self.workspace = torch.empty(need, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        self._id = None
        dist = None
        if world > 1 or nccl_id is not None:      # world == 1 + id: the multi-rank path on one GPU
            if nccl_id is None or len(nccl_id) != 128:
                raise SpfomError(1, "world > 1 needs the 128-byte nccl_id from rank 0")
            self._id = C.create_string_buffer(nccl_id, 128)
            dist = _Dist(int(rank), int(world), C.cast(self._id, C.c_void_p))
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(L.spfom_create(C.byref(self._inst), C.byref(self._params), None if dist is None else C.byref(dist),
                                  C.c_void_p(self.stream.cuda_stream), C.c_void_p(aligned),
                                  C.c_size_t(int(nbytes.value)), C.byref(h)))
        self._h = h
        self.workspace_bytes = int(nbytes.value)

    # --- C-ABI mirrors -----------------------------------------------------
    def step(self, k: int = 1) -> None:
        _check(load_library().spfom_step(self._h, int(k)), self._h)

    def duals(self) -> np.ndarray:
        out = np.empty(self.n_duals)
        _check(load_library().spfom_duals(self._h, out.ctypes.data), self._h)
        return out

    def primal(self):
        y, y0 = np.empty(self.nnz), np.empty(self.m)
        _check(load_library().spfom_primal(self._h, y.ctypes.data, y0.ctypes.data), self._h)
        return y, y0

    def usage(self) -> np.ndarray:
        out = np.empty(self.N)
        _check(load_library().spfom_usage(self._h, out.ctypes.data), self._h)
        return out

    def averages(self):
        y, y0, e = np.empty(self.nnz), np.empty(self.m), np.empty(self.n_duals)
        _check(load_library().spfom_averages(self._h, y.ctypes.data, y0.ctypes.data, e.ctypes.data), self._h)
        return y, y0, e

    def objective(self) -> float:
        v = C.c_double()
        _check(load_library().spfom_objective(self._h, C.byref(v)), self._h)
        return v.value

    def residuals(self) -> dict:
        r = _Residuals()
        _check(load_library().spfom_residuals(self._h, C.byref(r)), self._h)
        return {n: getattr(r, n) for n, _t in _Residuals._fields_}

    def set_state(self, y=None, y0=None, eta=None, s_prev=None) -> None:
        arrs = [None if a is None else _f64(a) for a in (y, y0, eta, s_prev)]
        _check(load_library().spfom_set_state(self._h, *[None if a is None else a.ctypes.data for a in arrs]),
               self._h)

    def info(self) -> dict:
        r = _Info()
        _check(load_library().spfom_info(self._h, C.byref(r)), self._h)
        d = {n: getattr(r, n) for n, _t in _Info._fields_ if not n.startswith("bin_")}
        d["bins"] = [dict(G=r.bin_G[b], Q=r.bin_Q[b], segments=r.bin_segments[b]) for b in range(r.num_bins)]
        return d

    def time_kernels(self, iters: int):
        """(ms in the primal kernels, ms in the rest) summed over `iters` un-graphed iterations."""
        ms = np.zeros(2)
        _check(load_library().spfom_time_kernels(self._h, int(iters), ms.ctypes.data), self._h)
        return float(ms[0]), float(ms[1])

    def recover(self):
        """SBLP -> CBLP policy of the current iterate (spfom_recover): (order,
        alpha) -- per row, product ids by y/v descending and the probabilities
        of the nested assortments S_0..S_k (alpha row i at seg_ptr[i] + i)."""
        order = np.empty(self.nnz, dtype=np.int32)
        alpha = np.empty(self.nnz + self.m)
        _check(load_library().spfom_recover(self._h, order.ctypes.data, alpha.ctypes.data), self._h)
        return order, alpha

    def recover_timed(self) -> float:
        """Device milliseconds of the recovery kernels over the whole instance
        (spfom_recover_timed: same launches as recover(), no host copies)."""
        ms = np.zeros(2)
        _check(load_library().spfom_recover_timed(self._h, ms.ctypes.data), self._h)
        return float(ms[0])

    def step_timed(self, k: int):
        """k iterations (two graph replays each) with CUDA events around the
        primal kernels; returns (primal ms summed over the k iterations, total ms)."""
        ms = np.zeros(2)
        _check(load_library().spfom_step_timed(self._h, int(k), ms.ctypes.data), self._h)
        return float(ms[0]), float(ms[1])

    @property
    def iteration(self) -> int:
        return int(load_library().spfom_iteration(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            load_library().spfom_destroy(self._h)
            self._h = None
        self._placement_pad = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
