"""Newton passes of K1's projection under different warm starts, simulated on
the host from the GPU's own iterates (huge, converge preset).

The GPU run supplies y_t, y0_t, eta_t after every iteration t.  For a sample
of segments the script re-solves each iteration's projection (z_t = y_{t-1} +
theta (r - eta_{t-1}), z0 = y0_{t-1}) with a numpy replica of project_group's
schedule (FULL pass: classification, piece sums, R, J, Newton step with the
sufficient-decrease / halving rule; CHECK pass: re-classification only) and
counts passes per segment for warm starts
  prev     x_{t-1}                          (the kernel today)
  extrap   x_{t-1} + gamma (x_{t-1} - x_{t-2})
The replica's final y is compared with the GPU's (checks the replica).  Warp
cost ~ the max over the 8 segments of a warp round: reported as the mean of
per-8 maxima."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np

import bench
from paper_2602_22421_b200 import Params, Solver

T = int(os.environ.get("ITERS", "40"))
S = int(os.environ.get("SAMPLE", "16000"))
inst = bench.load_instance("huge", "/tmp/spfom_cache")
rng = np.random.default_rng(7)
segs = np.sort(rng.choice(inst.m, S, replace=False))
k = np.diff(inst.seg_ptr)
K = int(((k.max() + 3) // 4) * 4)
idx = np.full((S, K), -1, np.int64)
for r, i in enumerate(segs):
    a, b = inst.seg_ptr[i], inst.seg_ptr[i + 1]
    idx[r, :b - a] = np.arange(a, b)
mask = idx >= 0
ent = np.where(mask, idx, 0)
V = np.where(mask, inst.attract[ent], 0.0)
W = np.where(mask, inst.shadow[ent], 0.0)
OM = np.where(mask, W / np.where(mask, V, 1.0), 0.0)
PJ = np.where(mask, inst.prod_idx[ent], 0)
LAM = inst.arrival[segs]
VT0 = inst.no_purchase[segs] + W.sum(1)
SVT = (V - W).sum(1)
R_ = inst.price

p = Params.converge()
theta = p.theta
s = Solver(inst, p)
Ys, Y0s, ETAs = [], [], []
y, y0 = s.primal()
Ys.append(np.where(mask, y[ent], 0.0)); Y0s.append(y0[segs].copy()); ETAs.append(s.duals().copy())
for t in range(T):
    s.step(1)
    y, y0 = s.primal()
    Ys.append(np.where(mask, y[ent], 0.0)); Y0s.append(y0[segs].copy()); ETAs.append(s.duals().copy())
s.close()


def project(z, z0, x):
    """numpy replica of project_group (per segment); returns y, y0, x, passes"""
    x0, x1, x2 = x[:, 0].copy(), x[:, 1].copy(), x[:, 2].copy()
    n = z.shape[0]
    tol = 1e-13 * (LAM + np.abs(z0) + np.abs(z).sum(1)) * np.maximum(1.0, VT0)
    a0, a1, a2 = x0.copy(), x1.copy(), x2.copy()
    d0 = np.zeros(n); d1 = np.zeros(n); d2 = np.zeros(n)
    step = np.ones(n); Ra = np.zeros(n)
    cA = np.zeros(z.shape, bool); fA = np.zeros(z.shape, bool)
    go = np.ones(n, bool); full = np.ones(n, bool); first = np.ones(n, bool)
    passes = np.zeros(n, np.int64)
    for _ in range(200):
        if not go.any():
            break
        a = OM * x1[:, None] + (z - x0[:, None])
        cap = V * x2[:, None]
        C = a >= cap
        F = ~C & (a > 0.0)
        chk = go & ~full
        changed = ((C != cA) | (F != fA)).any(1)
        passes[go] += 1
        done_chk = chk & ~changed
        go[done_chk] = False
        full[chk & changed] = True
        fu = go & full & ~chk
        if fu.any():
            vc = np.where(C, V, 0.0); af = np.where(F, a, 0.0); wf = np.where(F, OM, 0.0)
            rva = (vc * a).sum(1); cv = vc.sum(1); cvw = (vc * OM).sum(1); cvv = (vc * V).sum(1)
            sfa = af.sum(1); sfwa = (OM * af).sum(1); fw = wf.sum(1); fww = (wf * OM).sum(1); nf = F.sum(1)
            y0c = z0 - x0 + x1
            R0 = rva - x2 * cvv - VT0 * x1
            R1 = y0c + x2 * cvw + sfwa - VT0 * x2
            R2 = y0c + x2 * cv + sfa - LAM
            nr = np.maximum(np.abs(R0), np.maximum(np.abs(R1), np.abs(R2)))
            done = fu & ~(nr > tol)
            go[done] = False
            act = fu & ~done
            acc = act & (first | (nr <= (1.0 - 1e-4 * step) * Ra))
            back = act & ~acc
            if acc.any():
                J = np.zeros((n, 3, 3))
                J[:, 0, 0] = -cv; J[:, 0, 1] = cvw - VT0; J[:, 0, 2] = -cvv
                J[:, 1, 0] = -1.0 - fw; J[:, 1, 1] = 1.0 + fww; J[:, 1, 2] = cvw - VT0
                J[:, 2, 0] = -1.0 - nf; J[:, 2, 1] = 1.0 + fw; J[:, 2, 2] = cv
                Rv = np.stack([R0, R1, R2], 1)
                ii = np.where(acc)[0]
                d = -np.linalg.solve(J[ii], Rv[ii][:, :, None])[:, :, 0]
                a0[ii], a1[ii], a2[ii] = x0[ii], x1[ii], x2[ii]
                d0[ii], d1[ii], d2[ii] = d[:, 0], d[:, 1], d[:, 2]
                Ra[ii] = nr[ii]
                cA[ii] = C[ii]; fA[ii] = F[ii]
                step[ii] = 1.0
                full[ii] = False
            step[back] *= 0.5
            full[back] = True
            x0 = np.where(act, a0 + step * d0, x0)
            x1 = np.where(act, a1 + step * d1, x1)
            x2 = np.where(act, a2 + step * d2, x2)
            first[act] = False
    a = OM * x1[:, None] + (z - x0[:, None])
    cap = V * x2[:, None]
    yv = np.where(a >= cap, cap, np.where(a > 0.0, a, 0.0))
    return yv, z0 - x0 + x1, np.stack([x0, x1, x2], 1), passes


def run(policy, gamma=1.0):
    x = np.stack([np.zeros(S), np.zeros(S), LAM / (VT0 + SVT)], 1)
    xprev = x.copy()
    stats = []
    worst = 0.0
    for t in range(1, T + 1):
        g = R_[PJ] - ETAs[t - 1][PJ]
        z = np.where(mask, Ys[t - 1] + theta * g, 0.0)
        z0 = Y0s[t - 1]
        if policy == "extrap" and t >= 3:
            xw = x + gamma * (x - xprev)
            xw[:, 2] = np.maximum(xw[:, 2], 0.5 * x[:, 2])
        else:
            xw = x
        yv, y0n, xn, ps = project(z, z0, xw)
        worst = max(worst, float(np.abs(np.where(mask, yv, 0.0) - Ys[t]).max() / max(1.0, np.abs(Ys[t]).max())))
        xprev, x = x, xn
        n8 = (S // 8) * 8
        stats.append((t, ps.mean(), (ps > 2).mean(), ps[:n8].reshape(-1, 8).max(1).mean()))
    return stats, worst


for pol, gam in (("prev", 0.0), ("extrap", 1.0), ("extrap", 0.5)):
    st, worst = run(pol, gam)
    print(f"== warm start {pol} gamma {gam}: replica vs GPU y max rel diff {worst:.2e}")
    for (t, m_, p2, w8) in st:
        if t in (1, 2, 3, 5, 8, 10, 15, 20, 25, 30, 35, 40):
            print(f"  iteration {t:3d}: passes {m_:.3f}  P(>2) {p2:.3f}  warp max {w8:.3f}")
    sel = [r for r in st if 6 <= r[0] <= 25]
    if sel:
        print(f"  iterations 6-25: passes {np.mean([r[1] for r in sel]):.3f}  warp max {np.mean([r[3] for r in sel]):.3f}")
    sys.stdout.flush()
