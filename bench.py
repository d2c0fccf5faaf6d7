#!/usr/bin/env python
"""SPFOM iteration throughput on B200 (BASELINE.json metric: SPFOM iterations/s
and nnz/s, fp64, % of the HBM roofline).

One step = one SPFOM iteration (primal projection of every
segment, usage reduction A y, NCCL allreduce when N > 1, dual step) over the
BASELINE "huge" config (m = 1e6 segments, N = 1e5 products, 50M variables),
converge preset.  Contract and definitions: DESIGN.md §Measurement.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Eager CUDA module loading (read at CUDA initialisation, so before torch
# touches the GPU).  Measured on B200 (round 2): in the first iterations (the
# bench window) K1 is the same with lazy and eager loading (0.444 ms), but
# after ~1500 iterations it is 0.498 ms with lazy loading against 0.441 ms
# eager (profiles/r02_placement.txt).  An explicit setting in the
# environment wins.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

METRIC = "SPFOM iterations/s (fp64, full sweep)"
UNIT = "iterations/s"
BYTES_PER_NNZ = 36        # prod_idx 4 + v 8 + omega 8 + y read 8 + y write 8
BYTES_PER_SEGMENT = 36    # offset 4 + lambda 8 + vt0 8 + y0 read/write 16
BYTES_PER_PRODUCT = 72    # K3: s, s_prev, eta, c, tau, r read; eta, g, s_prev write


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="huge")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-iters", type=int, default=50, help="unused (kept for old command lines)")
    ap.add_argument("--cache", default=None, help="directory to cache the generated instance (npz)")
    ap.add_argument("--mode", default="throughput", choices=["throughput", "ttg", "features"],
                    help="ttg: time-to-gap of the full sweep vs sampled blocks B = m/2^k (SURVEY 8(f) rank 1); "
                         "features: device throughput of the a8 / 8(f) rows (averaging, paper preset full and "
                         "sampled, bundles, recovery) on --config")
    ap.add_argument("--stacked", action="store_true",
                    help="multi-period configs: pass the stacked instance as one period (no shared structure)")
    return ap.parse_args()


def load_instance(name: str, cache):
    from spfom_inputs import Instance, generate

    if not cache:
        return generate(name)
    import numpy as np

    path = os.path.join(cache, f"{name}.npz")
    if os.path.exists(path):
        z = np.load(path, allow_pickle=True)
        return Instance(name, z["seg_ptr"], z["prod_idx"], z["attract"], z["shadow"], z["no_purchase"],
                        z["arrival"], z["price"], z["capacity"], z["present"], z["meta"].item())
    inst = generate(name)
    os.makedirs(cache, exist_ok=True)
    np.savez(path, seg_ptr=inst.seg_ptr, prod_idx=inst.prod_idx, attract=inst.attract, shadow=inst.shadow,
             no_purchase=inst.no_purchase, arrival=inst.arrival, price=inst.price, capacity=inst.capacity,
             present=inst.present, meta=np.array(inst.meta, dtype=object))
    return inst


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload: str, kernel="k_primal"):
    """dram read+write bytes per launch of the dominant kernel from the committed
    ncu --set full summary (profiles/ncu_summary.json) of THIS workload, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        e = d.get(kernel if workload == "huge" else f"{kernel}@{workload}", {})
        if e.get("workload", "huge") != workload or not e.get("covers_k1", True):
            return None
        return e.get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_info():
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = "unknown"
    return model, os.cpu_count()


# --------------------------------------------------------------------- oracle legs
def oracle_sample_rate(inst, seconds_budget: float, label: str):
    """The CPU oracle (single thread, as it stands) on a leading-segment sample
    of `inst`; returns (iterations/s scaled to the full instance, description)."""
    import oracle

    probe_segs = min(inst.m, 2000)
    sub = inst.segment_slice(0, probe_segs)
    S = oracle.OracleSolver(sub)
    t0 = time.perf_counter()
    S.step()
    per_nnz = (time.perf_counter() - t0) / max(sub.nnz, 1)
    # choose the sample so that `iters` iterations take about the budget
    iters = 3
    target_nnz = seconds_budget / iters / max(per_nnz, 1e-12)
    segs = int(min(inst.m, max(probe_segs, target_nnz / max(inst.nnz / inst.m, 1))))
    sub = inst.segment_slice(0, segs)
    S = oracle.OracleSolver(sub)
    t0 = time.perf_counter()
    for _ in range(iters):
        S.step()
    dt = (time.perf_counter() - t0) / iters
    frac = sub.nnz / inst.nnz
    rate = frac / dt
    desc = (f"{label}: oracle/spfom_oracle.c (gcc -O2, 1 thread) on the first {segs} of {inst.m} segments "
            f"({sub.nnz} of {inst.nnz} nnz, all {inst.N} products), {iters} full-sweep iterations, "
            f"{dt * 1e3:.1f} ms/iteration; iterations/s scaled by the nnz fraction {frac:.4g}")
    return rate, desc, 1


def run_reference(args, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host cores."""
    if rank != 0:
        return
    from spfom_inputs import generate

    inst = load_instance(args.config, args.cache)
    # size each step so that warmup + steps finish within ~3 minutes
    budget_per_step = min(1.0, 150.0 / max(1, args.steps + args.warmup))
    import oracle

    probe = inst.segment_slice(0, min(inst.m, 2000))
    S = oracle.OracleSolver(probe)
    t0 = time.perf_counter()
    S.step()
    per_nnz = (time.perf_counter() - t0) / max(probe.nnz, 1)
    segs = int(min(inst.m, max(50, budget_per_step / per_nnz / max(inst.nnz / inst.m, 1))))
    sub = inst.segment_slice(0, segs)
    S = oracle.OracleSolver(sub)
    for _ in range(args.warmup):
        S.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        S.step()
    dt = time.perf_counter() - t0
    frac = sub.nnz / inst.nnz
    value = args.steps * frac / dt
    model, ncpu = cpu_info()
    sample = (f"each step = one oracle full-sweep iteration over the first {segs} of {inst.m} segments "
              f"({sub.nnz} nnz, all {inst.N} products); iterations/s scaled by the nnz fraction {frac:.4g}; "
              f"host {model}, {ncpu} logical CPUs, 1 used")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(inst, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "nnz_per_s": value * inst.nnz}
    print(json.dumps(line), flush=True)


def workload_config(inst, world):
    T = int(inst.meta.get("T", 1))
    extra = {"periods": T, "layout": "shared structure (num_periods = T)"} if T > 1 else {}
    return {"workload": inst.name, "m": inst.m, "N": inst.N, "nnz": inst.nnz, **extra, "preset": "converge",
            "theta": 1.0, "tau": "0.9/n_j", "extrapolation": 1.0, "mu": 0.0, "block": "full sweep",
            "parallelism": f"segments sharded over {world} GPU(s) by nnz; NCCL allreduce of s each iteration"
            if world > 1 else "1 GPU",
            "l2": "no flush: per-iteration working set 1.8 GB >> 126 MB L2" if inst.nnz > 10_000_000 else
            "working set fits L2 (no flush)",
            "cuda_module_loading": os.environ.get("CUDA_MODULE_LOADING", "LAZY")}


# --------------------------------------------------------------------- time to gap
def run_ttg(args):
    """Converge preset, full sweep (B = m) vs pre-generated sampled blocks
    B = m/2, m/4, m/8: iterations and device time (CUDA events around the
    steps only; residual checks every 50 m/B iterations are outside the timed
    spans) until max(|rel_gap|, infeas_rel) <= 1e-3 / 1e-4 / 1e-6."""
    import torch

    from paper_2602_22421_b200 import Params, Solver
    from spfom_inputs import block_sequence

    inst = load_instance(args.config, args.cache)
    m = inst.m
    stream_results = []
    for frac in (1, 2, 4, 8):
        B = m // frac
        blocks = None if frac == 1 else block_sequence(m, B, 512, 11)
        s = Solver(inst, Params.converge(blocks=blocks))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev_ms, it, hist = 0.0, 0, []
        for _ in range(400):
            e0.record(s.stream)
            s.step(50 * frac)
            e1.record(s.stream)
            torch.cuda.synchronize()
            dev_ms += e0.elapsed_time(e1)
            it += 50 * frac
            r = s.residuals()
            hist.append((it, dev_ms, max(abs(r["rel_gap"]), r["infeas_rel"])))
            if hist[-1][2] <= 1e-6:
                break
        first = lambda th: next(({"iters": i, "ms": round(t, 3)} for i, t, g in hist if g <= th), None)
        stream_results.append({"B": B, "exec": "persistent (k_small)" if s.info()["persistent"] else "graph",
                               "ttg_1e-3": first(1e-3), "ttg_1e-4": first(1e-4), "ttg_1e-6": first(1e-6),
                               "final_gap": hist[-1][2], "iterations": hist[-1][0],
                               "ms_per_iteration": hist[-1][1] / hist[-1][0]})
        s.close()
    print(json.dumps({"mode": "time-to-gap", "config": workload_config(inst, 1), "unit": "ms (device, CUDA events)",
                      "preset": "converge (theta 1, tau_j 0.9/n_j, extrapolation 1)", "results": stream_results}),
          flush=True)


# --------------------------------------------------------------------- feature rows
def run_features(args):
    """One JSON line per row: iterations/s (CUDA events over `steps` timed
    iterations after `warmup`, step_timed) and K1's share, for the converge
    preset with and without averaging (a8), the paper preset (theta = inf exact
    argmax, tau 0.1) full sweep and with sampled blocks B = m/4 (8(f) 1), the
    NRM bundle instance (8(f) 3); then the device time of the SBLP -> CBLP
    recovery of the converged iterate (8(f) 2)."""
    import torch

    from paper_2602_22421_b200 import Params, Solver
    from spfom_inputs import block_sequence, with_bundles

    inst = load_instance(args.config, args.cache)
    peak, peak_src = measured_peaks()
    steps, warm = max(1, min(args.steps, 500)), max(3, args.warmup)
    m = inst.m
    rows = [("converge", inst, Params.converge()),
            ("converge + averaging (a8)", inst, Params.converge(averaging=True)),
            ("paper preset, full sweep (theta = inf)", inst, Params.paper()),
            ("paper preset, sampled B = m/4 (8(f) 1)", inst, Params.paper(blocks=block_sequence(m, m // 4, 64, 5)))]
    if int(inst.meta.get("T", 1)) > 1:
        rows.pop()            # sampled blocks are rejected with shared periods (spfom.h)
    t0 = time.perf_counter()
    binst = with_bundles(inst, seed=3)
    rows.append((f"bundles / NRM, L = {binst.num_resources} resources (8(f) 3)", binst, Params.converge()))
    gen_s = time.perf_counter() - t0
    for label, ins, prm in rows:
        s = Solver(ins, prm)
        s.step(warm)
        torch.cuda.synchronize()
        k1, tot = s.step_timed(steps)
        line = {"mode": "features", "row": label, "config": workload_config(ins, 1),
                "value": steps / (tot / 1e3), "unit": "iterations/s", "steps": steps, "warmup": warm,
                "ms_per_step": tot / steps, "k1_ms_avg": k1 / steps, "k1_share": k1 / tot,
                "exec": "persistent (k_small)" if s.info()["persistent"] else "graph",
                "launches_per_iteration": int(s.info()["launches_per_iteration"])}
        if "bundles" in label:
            line["bundle_generation_s"] = gen_s
        if label == "converge":
            s.step(max(0, 1000 - warm - steps))
            ms = s.recover_timed()
            nnz, T = ins.nnz, int(ins.meta.get("T", 1))
            # algorithmic bytes: per entry id 4 + v 8 + omega 8 + y 8 + original id 4 read, order 4 + alpha 8
            # written; per segment qoff 4 + (lambda, vt0) 16 + y0 8 read, alpha_0 8 written
            rb = 44 * nnz + 36 * ins.m
            print(json.dumps({"mode": "features", "row": "SBLP -> CBLP recovery (8(f) 2)",
                              "config": workload_config(ins, 1), "iteration": s.iteration,
                              "value": ins.m / (ms / 1e3), "unit": "segments/s", "ms": ms,
                              "roofline": {"bound": "hbm", "achieved": rb / (ms / 1e3) / 1e9, "peak": peak,
                                           "unit": "GB/s", "frac": rb / (ms / 1e3) / 1e9 / peak,
                                           "bytes": rb, "bytes_rule": "44 B/nnz + 36 B/segment",
                                           "peak_source": peak_src},
                              "note": "device time of every k_recover launch (CUDA events, no host copies); "
                                      "rank-by-counting sort per segment, so ALU-heavy for long rows"}),
                  flush=True)
        s.close()
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU arm
def main():
    args = parse_args()
    if args.mode == "ttg":
        run_ttg(args)
        return
    if args.mode == "features":
        run_features(args)
        return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus == 1 else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2602_22421_b200 import Params, Solver, nccl_unique_id, partition
    from spfom_inputs import generate

    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    inst = load_instance(args.config, args.cache)
    T = int(inst.meta.get("T", 1))
    if T > 1:
        # multi-period: whole base segments (all T periods) per rank, shared structure
        from spfom_inputs import period_slice
        mb = int(inst.meta.get("m_per_period", inst.m // T))
        bounds = partition(inst.seg_ptr[: mb + 1], world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        shard = period_slice(inst, lo, hi) if world > 1 else inst
    else:
        bounds = partition(inst.seg_ptr, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        shard = inst.segment_slice(lo, hi) if world > 1 else inst
    nid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    params = Params.converge()
    pad = 0   # no placement pad: the workspace offset does not change K1 (profiles/r02_placement.txt)
    kw = dict(device=device, rank=rank, world=world, nccl_id=nid, segment_offset=lo,
              num_segments_global=inst.m if T == 1 else int(inst.meta.get("m_per_period", inst.m // T)),
              shared_periods=not args.stacked, workspace_offset_bytes=pad)
    if args.stacked:
        T = 1

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    solver = Solver(shard, params, **kw)
    info = solver.info()
    stream = solver.stream

    # warm-up (graph replays)
    solver.step(args.warmup)
    torch.cuda.synchronize(device)

    # timed region: exactly K iterations, barrier + sync on both sides
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize(device)
    ev0.record(stream)
    # each iteration = one replay of the iteration graph (4 iterations per graph
    # launch), whose event-record nodes bracket the primal kernels on the
    # solver's stream (roofline.achieved is live, over this region).  The
    # region is the device time from the first iteration's first event to the
    # event recorded after the last iteration (region_ms); ev0 / ev1 around
    # the call also contain the host's event bookkeeping inside step_timed.
    primal_ms_sum, region_ms = solver.step_timed(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize(device)
    barrier()
    ms_outer = ev0.elapsed_time(ev1)
    clocks = sampler.stop()
    ms = max_over_ranks(region_ms)
    value = args.steps / (ms / 1e3)
    k1_ms = max_over_ranks(primal_ms_sum) / args.steps
    rest_ms = max(0.0, ms / args.steps - k1_ms)
    res = solver.residuals()
    solver.close()

    peak, peak_src = measured_peaks()
    # algorithmic K1 bytes: structure (ids 4 + v 8 + omega 8) once per base entry, y r/w 16 per
    # (period) entry; offset 4 per base segment, lambda 8 + vt0 8 + y0 r/w 16 per (period) segment
    # (T = 1: 36 B/nnz + 36 B/segment)
    k1_bytes = 20 * shard.nnz // T + 16 * shard.nnz + 4 * shard.m // T + 32 * shard.m
    k1_achieved = k1_bytes / (k1_ms / 1e3) / 1e9
    iter_bytes = (20 * inst.nnz // T + 16 * inst.nnz + 4 * inst.m // T + 32 * inst.m) + BYTES_PER_PRODUCT * inst.N
    traffic = ncu_traffic(args.config)

    # e2e through the public API with host buffers: create (H2D) + K steps + duals/primal (D2H)
    # (three independent repetitions, each from the host arrays; the median is reported)
    e2e_reps = []
    for _ in range(3):
        barrier()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        s2 = Solver(shard, params, **kw)
        s2.step(args.steps)
        eta = s2.duals()
        y, y0 = s2.primal()
        t1 = time.perf_counter()
        e2e_info = s2.info()
        s2.close()
        del eta, y, y0
        e2e_reps.append(max_over_ranks(t1 - t0))
    e2e_s = sorted(e2e_reps)[1]
    e2e_value = args.steps / e2e_s
    nq = e2e_info["nnz_padded"] // 4
    h2d = nq * (16 + 32 + 32) + (shard.m + 1) * 4 + shard.m * (16 + 8 + 32 + 4) + (shard.N + 1) * 8 * 4
    d2h = shard.N * 8 + nq * 32 + shard.m * 8

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, desc, cores = oracle_sample_rate(inst, 15.0, "GPU-arm cpu_baseline")
        model, ncpu = cpu_info()
        cpu_baseline = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                        "sample": desc + f"; host {model}, {ncpu} logical CPUs"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(inst, world), workspace_offset_gib=pad >> 30),
            "nnz_per_s": value * inst.nnz,
            "iteration_hbm": {"canonical_bytes": iter_bytes,
                              "achieved_gbs": iter_bytes * value / 1e9,
                              "frac_of_measured": iter_bytes * value / 1e9 / peak,
                              "frac_of_8tbs": iter_bytes * value / 1e9 / 8000.0},
            "roofline": {"bound": "hbm", "kernel": "k_primal (K1: gather + gradient step + projection + A y scatter)",
                         "achieved": k1_achieved, "peak": peak, "unit": "GB/s", "frac": k1_achieved / peak,
                         "traffic": traffic, "bytes_per_launch": k1_bytes,
                         "bytes_rule": (f"{BYTES_PER_NNZ} B/nnz x {shard.nnz} + {BYTES_PER_SEGMENT} B/segment x {shard.m}"
                                        if T == 1 else
                                        f"20 B/base nnz x {shard.nnz // T} + 16 B/nnz x {shard.nnz} + "
                                        f"4 B/base segment x {shard.m // T} + 32 B/segment x {shard.m} (T = {T} shared)"),
                         "k1_ms_avg": k1_ms, "rest_ms_avg": rest_ms, "k1_share_of_step": k1_ms / (ms / args.steps),
                         "k1_timing": ("CUDA event-record nodes around the primal kernels of every timed iteration "
                                       "(solver stream, inside the iteration graph)"
                                       if not info.get("persistent") else
                                       "persistent small-regime kernel (whole iterations): CUDA events around all of them"),
                         "peak_source": peak_src, "frac_of_8tbs": k1_achieved / 8000.0},
            "clocks": clocks,
            "timed_region": {"device_ms": ms, "outer_events_ms": ms_outer,
                             "note": "value = steps / device_ms: events on the solver stream from the first "
                                     "iteration's start to the end of the last; outer_events_ms (events around "
                                     "the step_timed call) also holds its host-side event bookkeeping"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / args.steps,
                    "d2h_bytes_per_step": d2h / args.steps,
                    "definition": "wall time of Solver(host arrays) [validate+layout+H2D] + K graph-replayed "
                                  "iterations + duals()+primal() D2H, through the C ABI; median of 3 repetitions",
                    "reps_s": [round(x, 4) for x in e2e_reps]},
            "gpu_launches": int(info["launches_per_iteration"]) * args.steps,
            "cpu_baseline": cpu_baseline,
            "residuals_after": {k: res[k] for k in ("iteration", "rel_gap", "infeas_rel", "newton_failures",
                                                    "newton_restarts")},
            "newton_passes_per_segment_iteration": res["newton_passes"] / max(1, res["iteration"] * shard.m),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
