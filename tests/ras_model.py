"""TEST MODEL of the distributed GMRES engine (csrc/cuda/gmres_engine.cu) for the
CPU suite: the same algorithm -- reference gmres.cpp:28-137 control flow and
Givens arithmetic, CGS2 orthogonalisation with two all-reduces per iteration,
halo exchanges before the local apply and the local SpMV -- in numpy, with the
local work done by the C oracle and the collectives by a torch.distributed
(gloo) group. It checks, on CPU with world sizes > 1, that the product's C++
RAS plan (hec_ras_plan_create) plus this algorithm reproduce the reference:
the distributed apply bitwise, GMRES iterations within +-1.
"""
import math

import numpy as np

from oracle.oracle import Csr


class GlooComm:
    def __init__(self, plan):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.plan = torch, dist, plan
        self.allreduces = self.exchanges = 0

    def allreduce(self, arr):
        if self.plan.world == 1:
            return arr
        self.allreduces += 1
        t = self.torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
        self.dist.all_reduce(t)
        return t.numpy()

    def exchange(self, vloc):
        p = self.plan
        if p.world == 1:
            return
        self.exchanges += 1
        send = self.torch.from_numpy(np.ascontiguousarray(vloc[:p.n_own][p.send_idx]))
        recv = self.torch.empty(p.n_loc - p.n_own, dtype=self.torch.float64)
        self.dist.all_to_all_single(recv, send, p.recv_counts, p.send_counts)
        vloc[p.n_own:] = recv.numpy()


class OracleLocal:
    """Rank-local operator: the oracle's ILU(0) apply of the block and the local SpMV rows."""

    def __init__(self, H, a, plan, orc):
        self.orc, self.plan = orc, plan
        f = H.ilu0(H.csr_submatrix(a, plan.ext))
        self.pl = orc.prepare(Csr.of(f.l))
        self.pu = orc.prepare(Csr.of(f.u), upper=True)
        self.owned = (plan.out_index >= 0).astype(np.int8)
        A = Csr.of(a)
        loc = np.full(a.n_rows, -1, np.int64)
        loc[plan.own] = np.arange(plan.n_own)
        loc[plan.halo] = plan.n_own + np.arange(len(plan.halo))
        rp, ci, v = [0], [], []
        for r in plan.own:
            s, e = A.rp[r], A.rp[r + 1]
            ci.extend(loc[A.ci[s:e]].tolist())
            v.extend(A.v[s:e].tolist())
            rp.append(len(ci))
        self.A = Csr(plan.n_own, plan.n_loc, np.array(rp), np.array(ci), np.array(v))

    def apply(self, vloc):
        x = self.orc.apply(self.plan.n_loc, self.plan.gather, self.owned, self.pl, self.pu, vloc)
        return x[:self.plan.n_own]

    def matvec(self, zloc):
        return self.orc.spmv(self.A, zloc)


def gmres(local, comm, plan, b_own, restart=20, max_iters=10000, rel_tol=1e-6, abs_tol=0.0):
    n, nl, mr = plan.n_own, plan.n_loc, restart

    def norm(v):
        return math.sqrt(float(comm.allreduce(np.array([np.dot(v, v)]))[0]))

    def op(v_own):
        vloc = np.zeros(nl)
        vloc[:n] = v_own
        comm.exchange(vloc)
        zloc = np.zeros(nl)
        zloc[:n] = local.apply(vloc)
        comm.exchange(zloc)
        return local.matvec(zloc)

    bnorm = norm(b_own)
    threshold = max(rel_tol * bnorm, abs_tol)
    V = np.zeros((mr + 1, n))
    h = np.zeros((mr + 1, mr))
    cs, sn, g, y = np.zeros(mr), np.zeros(mr), np.zeros(mr + 1), np.zeros(mr)
    x = np.zeros(n)
    r = b_own.copy()
    rnorm, stalled, iters, converged = bnorm, False, 0, False
    while True:
        if rnorm <= threshold:
            converged = True
            break
        if iters >= max_iters or stalled:
            break
        V[0] = r / rnorm
        g[:] = 0.0
        g[0] = rnorm
        j, lucky = 0, False
        while j < mr and iters < max_iters:
            w = op(V[j])
            h1 = comm.allreduce(V[:j + 1] @ w)                       # CGS2 pass 1
            w = w - h1 @ V[:j + 1]
            red = comm.allreduce(np.concatenate([V[:j + 1] @ w, [np.dot(w, w)]]))  # pass 2 + ||w'||^2
            h2, ww = red[:j + 1], red[j + 1]
            hjj1 = math.sqrt(max(ww - float(np.dot(h2, h2)), 0.0))
            if hjj1 > 1e-300:
                V[j + 1] = (w - h2 @ V[:j + 1]) / hjj1
            else:
                lucky = True
            h[:j + 1, j] = h1 + h2
            h[j + 1, j] = hjj1
            for i in range(j):
                hi, hi1 = h[i, j], h[i + 1, j]
                h[i, j] = cs[i] * hi + sn[i] * hi1
                h[i + 1, j] = -sn[i] * hi + cs[i] * hi1
            denom = math.hypot(h[j, j], hjj1)
            cs[j], sn[j] = (h[j, j] / denom, hjj1 / denom) if denom > 0.0 else (1.0, 0.0)
            h[j, j], h[j + 1, j] = denom, 0.0
            gj = g[j]
            g[j], g[j + 1] = cs[j] * gj, -sn[j] * gj
            iters += 1
            j += 1
            if abs(g[j]) <= threshold or lucky:
                break
        for i in range(j - 1, -1, -1):
            s = g[i]
            for t in range(i + 1, j):
                s -= h[i, t] * y[t]
            y[i] = s / h[i, i]
        xc = y[:j] @ V[:j] if j else np.zeros(n)
        vloc = np.zeros(nl)
        vloc[:n] = xc
        comm.exchange(vloc)
        x = x + local.apply(vloc)
        xloc = np.zeros(nl)
        xloc[:n] = x
        comm.exchange(xloc)
        r = b_own - local.matvec(xloc)
        rn = norm(r)
        if lucky and rn > threshold:
            stalled = True
        rnorm = rn
    return x, dict(converged=converged, iterations=iters, rel=rnorm / bnorm if bnorm > 0 else rnorm,
                   allreduces=comm.allreduces, exchanges=comm.exchanges)
