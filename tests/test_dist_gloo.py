"""Multi-rank host logic on CPU (torch.distributed gloo, world_size 2 and 3).

The N > 1 path (Alg. 3): each rank owns a contiguous
segment range from spfom_partition (the C library's host function), the
per-product step sizes tau_j = 0.9 / n_j use GLOBAL column counts (allreduced
once at create), and every iteration allreduces the usage vector before an
identical dual step on every rank -- or (variant "rs", the library's default
for world > 1) each rank updates the duals of its slice of the products and
the slices are all-gathered.  Here the ranks' primal steps are emulated
with the CPU oracle; the test checks partition invariance against the single-
process oracle and that the ranks' duals are bitwise identical.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, errq, variant="plain"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2602_22421_b200 import partition
        from spfom_inputs import generate, period_slice, with_bundles

        if variant == "multi":
            # shared-structure multi-period: ranks own whole base segments (all T periods)
            inst = generate("multi", m=300, N=200, k=(10, 60), T=3)
            T, mb = 3, 300
            bounds = partition(inst.seg_ptr[: mb + 1], world)
            lo, hi = int(bounds[rank]), int(bounds[rank + 1])
            shard = period_slice(inst, lo, hi)
            rows = [(t * mb + lo, t * mb + hi) for t in range(T)]
        else:
            inst = generate("medium", m=900, N=300, k=(20, 80))
            if variant == "bundles":
                inst = with_bundles(inst, L=90, seed=4)
            bounds = partition(inst.seg_ptr, world)
            lo, hi = int(bounds[rank]), int(bounds[rank + 1])
            shard = inst.segment_slice(lo, hi)
            rows = [(lo, hi)]

        # global column counts -> tau (what spfom_create does with an NCCL allreduce)
        cnt = torch.from_numpy(np.bincount(shard.prod_idx, minlength=inst.N).astype(np.int64))
        dist.all_reduce(cnt)
        n = cnt.numpy()
        assert np.array_equal(n, np.bincount(inst.prod_idx, minlength=inst.N))
        if variant == "bundles":      # per resource: n_l = sum_{j uses l} n_j (reading c17)
            nl = np.zeros(inst.num_resources, dtype=np.int64)
            for j in range(inst.N):
                nl[inst.bundle_res[inst.bundle_ptr[j]:inst.bundle_ptr[j + 1]]] += n[j]
            tau = np.where(nl > 0, 0.9 / np.maximum(nl, 1), 0.9)
        else:
            tau = np.where(n > 0, 0.9 / np.maximum(n, 1), 0.9)

        S = oracle.OracleSolver(shard)
        S.tau_j[:] = tau
        ref = oracle.OracleSolver(inst)
        ent = np.concatenate([np.arange(inst.seg_ptr[a], inst.seg_ptr[b]) for a, b in rows])
        seg = np.concatenate([np.arange(a, b) for a, b in rows])
        N = inst.N
        chunk = (N + 1 + world - 1) // world          # spfom.cu: h->chunk (ReduceScatter slices)
        plo = rank * chunk
        for _t in range(40):
            s = torch.from_numpy(S.primal_shard())
            dist.all_reduce(s)
            if variant == "rs":
                # ReduceScatter -> dual step on this rank's slice -> AllGather
                # (the library's default for world > 1; gloo has no
                # reduce_scatter, so the slice is cut from the allreduce)
                sl = slice(min(plo, N), min(plo + chunk, N))
                new = oracle.dual_step(S.eta[sl], s.numpy()[sl], S.s[sl], inst.capacity[sl], tau[sl], 0.0, 1.0)
                mine = torch.zeros(chunk, dtype=torch.float64)
                mine[: new.shape[0]] = torch.from_numpy(new)
                parts = [torch.zeros(chunk, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, mine)
                S.eta[:] = torch.cat(parts).numpy()[:N]
                S.s[:] = s.numpy()
            else:
                S.dual_apply(s.numpy())
            ref.step()
            scale = max(float(np.abs(ref.eta).max()), 1e-300)
            assert np.abs(S.eta - ref.eta).max() <= 1e-12 * max(scale, 1.0), "eta drifted from single-rank run"
            assert np.abs(S.y - ref.y[ent]).max() <= 1e-12 * max(1.0, np.abs(ref.y).max())
            assert np.abs(S.y0 - ref.y0[seg]).max() <= 1e-12 * float(inst.arrival.max())
        # every rank holds bitwise-identical duals
        mine = torch.from_numpy(S.eta.copy())
        gathered = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine)
        for other in gathered:
            assert torch.equal(other, mine)
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("world,variant", [(2, "plain"), (3, "plain"), (2, "bundles"), (3, "multi"), (2, "rs"),
                                           (3, "rs")])
def test_sharded_iteration_matches_single_rank(world, variant):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(world, _free_port(), errq, variant), nprocs=world, join=True,
                       start_method="spawn")
    assert errq.empty(), errq.get()


def test_partition_respects_block_offsets():
    """Sampled blocks use global ids; a rank keeps the ids inside its range and
    shifts them by its segment_offset (host logic of spfom_create)."""
    from paper_2602_22421_b200 import partition
    from spfom_inputs import block_sequence, generate
    inst = generate("small", m=500, N=100, k=(5, 30))
    bounds = partition(inst.seg_ptr, 2)
    blocks = block_sequence(inst.m, 64, 5, seed=1)
    parts = []
    for r in range(2):
        lo, hi = bounds[r], bounds[r + 1]
        parts.append([row[(row >= lo) & (row < hi)] - lo for row in blocks])
    for t in range(5):
        rebuilt = np.concatenate([parts[0][t] + bounds[0], parts[1][t] + bounds[1]])
        assert np.array_equal(rebuilt, blocks[t])
