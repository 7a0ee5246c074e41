"""Restricted Additive Schwarz on several GPUs: one subdomain per process.

Reference: hec::build_preconditioner(a, ras | bilu0, blocks, overlap) +
hec::apply + hec::gmres (proj/src/precond.cpp:74-145, proj/src/gmres.cpp:28-137,
proj/src/partition.cpp:28-107). The reference keeps every block in one address
space and assembles them into one block-diagonal factor; here rank g of a
`torch.distributed` group (one process per GPU, NCCL) owns block g:

* rows: part g of the reference's partition (`own`, ascending), plus the halo
  `ext_g ∪ cols(A[own, :]) \\ own` ordered by (owning rank, row);
* local vectors: `[own | halo]` in that order; the halo segment is filled by
  one all-to-all per exchange (NCCL send/recv of exactly the rows each peer
  needs, no full-vector traffic);
* preconditioner: ilu0 / ilu_k / ilut of extract_block(A, ext_g) (the
  reference's own per-block factorization), prepared and solved by this
  library's B200 kernels; the restricted scatter writes owned rows only. This
  equals the reference's assembled block-diagonal solve bitwise (levels are
  computed per row from in-block dependencies only);
* SpMV: A[own, :] with columns renumbered into `[own | halo]`, same storage
  order, so each row sum is bitwise the reference's spmv_csr row;
* GMRES: the reference's algorithm line for line; dot products are local
  fixed-order partials summed with one all-reduce each (the only results that
  differ from the reference in rounding, hence iteration counts within ±1).

The host logic (`RasPlan`, `gmres`) is backend-agnostic: `DeviceOps` runs the
local work through the C-ABI on the GPU; the CPU test-suite plugs in the
oracle to check the distributed logic with the gloo backend.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import api as H


# --------------------------------------------------------------- plan ----
@dataclass
class RasPlan:
    """Everything rank `rank` needs, derived deterministically from the global
    matrix on every rank (no communication during setup)."""
    n: int
    rank: int
    world: int
    part_of: np.ndarray                 # global row -> owning rank
    own: np.ndarray                     # ascending global rows owned here
    ext: np.ndarray                     # ascending extended rows (the block)
    halo: np.ndarray                    # global rows of the halo segment, by (owner, row)
    send_idx: List[np.ndarray]          # per peer: local own positions to send, peer's halo order
    recv_counts: List[int]              # per peer: halo entries received
    gather: np.ndarray                  # block row k -> local [own | halo] index
    out_index: np.ndarray               # block row k -> own position, or -1
    a_rp: np.ndarray                    # local SpMV rows (own) in CSR, columns in [own | halo]
    a_ci: np.ndarray
    a_v: np.ndarray

    @property
    def n_own(self) -> int:
        return int(self.own.shape[0])

    @property
    def n_loc(self) -> int:
        return int(self.own.shape[0] + self.halo.shape[0])


def make_plan(a: H.CsrMatrix, world: int, rank: int, overlap: int) -> RasPlan:
    """The reference partition (partition_graph + extend_overlap) and this rank's maps."""
    part_of, ext_parts = H.partition(a, world, overlap)
    rp, ci, v = a.row_offsets, a.col_indices, a.values
    n = a.n_rows
    owns = [np.flatnonzero(part_of == p).astype(np.int32) for p in range(world)]
    needs = []
    for p in range(world):
        own_p = owns[p]
        # column indices of the part's rows (vectorised CSR row gather)
        starts, ends = rp[own_p], rp[own_p + 1]
        lens = ends - starts
        take = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(int(lens.sum()))
        cols = ci[take]
        need = np.setdiff1d(np.union1d(ext_parts[p], cols), own_p)
        # halo order: by owning rank, then row (stable)
        order = np.lexsort((need, part_of[need]))
        needs.append(need[order].astype(np.int32))
    own = owns[rank]
    halo = needs[rank]
    loc = np.full(n, -1, dtype=np.int64)
    loc[own] = np.arange(own.size)
    loc[halo] = own.size + np.arange(halo.size)
    # what each peer needs from me, in the peer's halo order (already sorted by row)
    pos_in_own = np.full(n, -1, dtype=np.int64)
    pos_in_own[own] = np.arange(own.size)
    send_idx, recv_counts = [], []
    for p in range(world):
        if p == rank:
            send_idx.append(np.zeros(0, np.int64))
            recv_counts.append(0)
            continue
        mine = needs[p][part_of[needs[p]] == rank]
        send_idx.append(pos_in_own[mine])
        recv_counts.append(int(np.count_nonzero(part_of[halo] == p)))
    ext = ext_parts[rank].astype(np.int32)
    gather = loc[ext].astype(np.int32)
    out_index = np.where(part_of[ext] == rank, pos_in_own[ext], -1).astype(np.int32)
    # local SpMV: owned rows, same storage order, columns renumbered
    starts, ends = rp[own], rp[own + 1]
    lens = (ends - starts).astype(np.int64)
    take = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(int(lens.sum()))
    a_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    a_ci = loc[ci[take]].astype(np.int32)
    if (a_ci < 0).any():
        raise RuntimeError("ras plan: SpMV column outside own + halo")
    return RasPlan(n, rank, world, part_of, own, ext, halo, send_idx, recv_counts, gather, out_index,
                   a_rp, a_ci, v[take].astype(np.float64))


# --------------------------------------------------------------- comm ----
class TorchComm:
    """Sum all-reduce of device scalars and the halo all-to-all over a
    torch.distributed group (NCCL: device buffers directly; gloo: staged
    through host memory)."""

    def __init__(self, plan: RasPlan, device):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.plan = plan
        self.device = device
        self.staged = dist.is_initialized() and dist.get_backend() != "nccl"
        self.single = (not dist.is_initialized()) or dist.get_world_size() == 1
        self.send_counts = [int(s.shape[0]) for s in plan.send_idx]
        self.send_idx = torch.tensor(np.concatenate(plan.send_idx) if plan.send_idx else np.zeros(0),
                                     dtype=torch.int64, device=device)
        self.n_send = int(self.send_idx.shape[0])
        self.allreduces = 0
        self.exchanges = 0

    def allreduce(self, t):
        """In-place sum over ranks of a small device tensor."""
        if self.single:
            return t
        self.allreduces += 1
        if self.staged:
            h = t.cpu()
            self.dist.all_reduce(h)
            t.copy_(h)
        else:
            self.dist.all_reduce(t)
        return t

    def exchange(self, vloc):
        """Fill the halo segment of a local [own | halo] vector from the owners."""
        if self.single:
            return vloc
        self.exchanges += 1
        torch = self.torch
        n_own = self.plan.n_own
        send = vloc[:n_own].index_select(0, self.send_idx) if self.n_send else vloc.new_zeros(0)
        recv = vloc[n_own:]
        if self.staged:
            hs, hr = send.cpu(), torch.empty(recv.shape[0], dtype=recv.dtype)
            self.dist.all_to_all_single(hr, hs, self.plan.recv_counts, self.send_counts)
            recv.copy_(hr)
        else:
            out = torch.empty_like(recv)
            self.dist.all_to_all_single(out, send, self.plan.recv_counts, self.send_counts)
            recv.copy_(out)
        return vloc


# ---------------------------------------------------------- device ops ----
class DeviceOps:
    """Local work of one subdomain on the B200 through the C-ABI."""

    def __init__(self, a: H.CsrMatrix, plan: RasPlan, kind: str = "ilu0", fill_level: int = 1,
                 ilut_p: int = 7, ilut_tol: float = 0.1, device=None):
        import torch
        self.torch = torch
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.plan = plan
        block = H.csr_submatrix(a, plan.ext)
        if kind == "ilu0":
            f = H.ilu0(block)
        elif kind == "iluk":
            f = H.ilu_k(block, fill_level)
        elif kind == "ilut":
            f = H.ilut(block, ilut_p, ilut_tol)
        else:
            raise ValueError(f"unknown local factorization {kind!r}")
        self.pl, self.pu = H.prepare_lower(f.l), H.prepare_upper(f.u)
        self.m = H.DevicePrecond.create_local(plan.n_loc, plan.n_own, self.pl, self.pu, plan.gather, plan.out_index)
        aloc = H.CsrMatrix.from_arrays(plan.n_own, plan.n_loc, plan.a_rp, plan.a_ci, plan.a_v)
        self.spmv = H.DeviceSpmv(aloc)
        self.kr = H.Krylov(plan.n_own)
        self.stream = None

    def vec(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def apply(self, vloc, z_own):
        self.m.apply(vloc, z_own)

    def matvec(self, zloc, w_own):
        self.spmv.run(zloc, w_own)

    def mgs(self, w, v_prev, h_prev, v_next, out):
        self.kr.mgs(w, v_prev, h_prev, v_next, out)

    def scale(self, y, x, s):
        self.kr.scale(y, x, s)

    def combine(self, j, xc, V, ldv, y):
        self.kr.combine(j, xc, V, ldv, y)

    def add(self, x, d):
        self.kr.add(x, d)

    def sqrt(self, a, out):
        self.kr.sqrt(a, out)

    def to_host(self, t):
        return t.cpu().numpy()

    def copy(self, dst, src):
        dst.copy_(src)

    def residual(self, r, b, ax):
        """r = b - A x, one IEEE subtraction per row (gmres.cpp:19-24)."""
        self.torch.sub(b, ax, out=r)

    def from_host(self, arr):
        return self.torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64), device=self.device)

    def sub(self, V, i, ldv, n):
        """View of column i of a (m+1) x ldv basis."""
        return V[i * ldv:i * ldv + n]


# --------------------------------------------------------------- gmres ----
@dataclass
class RasReport:
    converged: bool = False
    iterations: int = 0
    final_relative_residual: float = 0.0
    solve_seconds: float = 0.0
    inner_residuals: List[float] = field(default_factory=list)
    allreduces: int = 0
    exchanges: int = 0


def gmres(ops, comm, plan: RasPlan, b_own, restart: int = 20, max_iters: int = 10000, rel_tol: float = 1e-6,
          abs_tol: float = 0.0, precondition: bool = True):
    """Right-preconditioned restarted GMRES(m), zero initial guess: the
    reference's gmres.cpp:28-137 with distributed vectors (own rows only)."""
    if restart < 1:
        raise ValueError("gmres: restart must be >= 1")
    if max_iters < 0 or rel_tol < 0 or abs_tol < 0:
        raise ValueError("gmres: invalid configuration")
    t0 = time.perf_counter()
    n, nl, mr = plan.n_own, plan.n_loc, restart
    ldv = (max(n, 1) + 3) // 4 * 4  # 32-byte aligned basis columns (vectorised Krylov kernels)
    V = ops.vec((mr + 1) * ldv)
    b = ops.from_host(b_own)
    x, r = ops.vec(n), ops.vec(n)
    vloc, zloc = ops.vec(nl), ops.vec(nl)
    z, w = ops.vec(n), ops.vec(n)
    hcol = ops.vec(mr + 3)
    scal = ops.vec(2)
    yv = ops.vec(mr + 1)
    rep = RasReport()

    def norm_into(vec, dst_sq, dst):
        ops.mgs(vec, None, None, vec, dst_sq)          # local ||v||^2
        comm.allreduce(dst_sq)
        ops.sqrt(dst_sq, dst)

    def op_apply(src_own, dst_own):
        """dst = A M^-1 src (or A src), with the two halo exchanges."""
        if precondition:
            ops.copy(vloc[:n], src_own)
            comm.exchange(vloc)
            ops.apply(vloc, z)
            ops.copy(zloc[:n], z)
        else:
            ops.copy(zloc[:n], src_own)
        comm.exchange(zloc)
        ops.matvec(zloc, dst_own)

    norm_into(b, scal[0:1], scal[1:2])
    bnorm = float(ops.to_host(scal)[1])
    threshold = max(rel_tol * bnorm, abs_tol)
    h = np.zeros((mr + 1, mr))
    cs, sn, g, y = np.zeros(mr), np.zeros(mr), np.zeros(mr + 1), np.zeros(mr)
    ops.copy(r, b)
    rnorm = bnorm
    stalled = False
    rn_dev = scal[1:2]
    while True:
        if rnorm <= threshold:
            rep.converged = True
            break
        if rep.iterations >= max_iters or stalled:
            break
        ops.scale(ops.sub(V, 0, ldv, n), r, rn_dev)
        g[:] = 0.0
        g[0] = rnorm
        j = 0
        lucky = False
        while j < mr and rep.iterations < max_iters:
            vj = ops.sub(V, j, ldv, n)
            op_apply(vj, w)
            # MGS (gmres.cpp:72-76): step i removes the (i-1) component, then dots with v_i
            for i in range(j + 1):
                ops.mgs(w, ops.sub(V, i - 1, ldv, n) if i else None, hcol[i - 1:i] if i else None,
                        ops.sub(V, i, ldv, n), hcol[i:i + 1])
                comm.allreduce(hcol[i:i + 1])
            ops.mgs(w, vj, hcol[j:j + 1], w, hcol[j + 2:j + 3])  # last removal + ||w||^2
            comm.allreduce(hcol[j + 2:j + 3])
            ops.sqrt(hcol[j + 2:j + 3], hcol[j + 1:j + 2])
            ops.scale(ops.sub(V, j + 1, ldv, n), w, hcol[j + 1:j + 2])
            hc = ops.to_host(hcol[:j + 2])
            h[:j + 1, j] = hc[:j + 1]
            hjj1 = float(hc[j + 1])
            h[j + 1, j] = hjj1
            if not (hjj1 > 1e-300):
                lucky = True
            for i in range(j):  # Givens (gmres.cpp:85-104)
                hi, hi1 = h[i, j], h[i + 1, j]
                h[i, j] = cs[i] * hi + sn[i] * hi1
                h[i + 1, j] = -sn[i] * hi + cs[i] * hi1
            hjj = h[j, j]
            denom = math.hypot(hjj, hjj1)
            if denom > 0.0:
                cs[j], sn[j] = hjj / denom, hjj1 / denom
            else:
                cs[j], sn[j] = 1.0, 0.0
            h[j, j] = denom
            h[j + 1, j] = 0.0
            gj = g[j]
            g[j] = cs[j] * gj
            g[j + 1] = -sn[j] * gj
            rep.iterations += 1
            j += 1
            est = abs(g[j])
            rep.inner_residuals.append(est)
            if est <= threshold or lucky:
                break
        for i in range(j - 1, -1, -1):  # back substitution (gmres.cpp:115-119)
            s = g[i]
            for t in range(i + 1, j):
                s -= h[i, t] * y[t]
            y[i] = s / h[i, i]
        ops.copy(yv[:max(j, 1)], ops.from_host(y[:max(j, 1)]))
        ops.combine(j, w, V, ldv, yv)
        if precondition:
            ops.copy(vloc[:n], w)
            comm.exchange(vloc)
            ops.apply(vloc, z)
            ops.add(x, z)
        else:
            ops.add(x, w)
        # r = b - A x (gmres.cpp:126-131)
        ops.copy(zloc[:n], x)
        comm.exchange(zloc)
        ops.matvec(zloc, w)
        ops.residual(r, b, w)
        norm_into(r, scal[0:1], rn_dev)
        rn = float(ops.to_host(scal)[1])
        if lucky and rn > threshold:
            stalled = True
        rnorm = rn
    rep.final_relative_residual = rnorm / bnorm if bnorm > 0.0 else rnorm
    rep.solve_seconds = time.perf_counter() - t0
    rep.allreduces, rep.exchanges = comm.allreduces, comm.exchanges
    return x, rep


class RasGmres:
    """RAS-preconditioned GMRES with one subdomain per process/GPU."""

    def __init__(self, a: H.CsrMatrix, overlap: int = 1, restart: int = 20, max_iters: int = 10000,
                 rel_tol: float = 1e-6, abs_tol: float = 0.0, local: str = "ilu0", fill_level: int = 1,
                 ilut_p: int = 7, ilut_tol: float = 0.1, device=None):
        import torch
        import torch.distributed as dist
        world = dist.get_world_size() if dist.is_initialized() else 1
        rank = dist.get_rank() if dist.is_initialized() else 0
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.plan = make_plan(a, world, rank, overlap)
        self.ops = DeviceOps(a, self.plan, local, fill_level, ilut_p, ilut_tol, self.device)
        self.comm = TorchComm(self.plan, self.device)
        self.cfg = dict(restart=restart, max_iters=max_iters, rel_tol=rel_tol, abs_tol=abs_tol)

    def solve(self, b_global):
        """b: global right-hand side (host); returns (x on owned rows (device), report)."""
        b_own = np.ascontiguousarray(np.asarray(b_global, dtype=np.float64)[self.plan.own])
        return gmres(self.ops, self.comm, self.plan, b_own, **self.cfg)
