"""Restricted Additive Schwarz on several GPUs: one subdomain per process.

Thin Python face of the library's C++ RAS layer (include/hecsolve_c.h section
3: hec_ras_plan_*, hec_ras_create / apply / gmres; csrc/host/ras_plan.cpp,
csrc/cuda/gmres_engine.cu, csrc/cuda/comm.cpp). Reference:
hec::build_preconditioner(a, ras, blocks, overlap) + hec::apply + hec::gmres
(proj/src/precond.cpp:74-145, proj/src/gmres.cpp:28-137,
proj/src/partition.cpp:28-107), with block g on rank g:

* rows: part g of the reference's partition (`own`, ascending), plus the halo
  `ext_g u cols(A[own, :]) \\ own` ordered by (owning rank, row);
* preconditioner: ilu0 / ilu_k / ilut of extract_block(A, ext_g), solved by the
  B200 kernels; the restricted scatter writes owned rows only -- rank g's rows
  of the reference's assembled apply, bit for bit;
* SpMV: A[own, :] with columns renumbered into [own | halo], storage order kept;
* GMRES: the device engine (two all-reduces and two halo exchanges per
  iteration, CGS2), iteration counts within +-1 of the reference.

Communication: NCCL (device buffers over NVLink) when torch.distributed runs the
nccl backend -- rank 0 makes the NCCL unique id, torch.distributed broadcasts
it --, host callbacks over the torch.distributed group otherwise (gloo: e.g.
several ranks sharing one GPU in the tests), nothing on one rank.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L
from . import api as H
from ._lib import lib

check = H.check


@dataclass
class RasPlan:
    """Rank `rank`'s maps (copies of the C++ plan, csrc/host/ras_plan.cpp)."""
    n: int
    rank: int
    world: int
    part_of: np.ndarray
    own: np.ndarray
    ext: np.ndarray
    halo: np.ndarray
    send_offsets: np.ndarray
    send_idx: np.ndarray
    recv_offsets: np.ndarray
    gather: np.ndarray
    out_index: np.ndarray

    @property
    def n_own(self) -> int:
        return int(self.own.shape[0])

    @property
    def n_loc(self) -> int:
        return int(self.own.shape[0] + self.halo.shape[0])

    @property
    def send_counts(self) -> List[int]:
        return np.diff(self.send_offsets).tolist()

    @property
    def recv_counts(self) -> List[int]:
        return np.diff(self.recv_offsets).tolist()


def _plan_from_handle(h) -> RasPlan:
    v = L.RasPlanView()
    check(lib.hec_ras_plan_view_get(h, C.byref(v)))

    def arr(p, n):
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.int32)

    w = v.world
    return RasPlan(v.n, v.rank, w, arr(v.part_of, v.n), arr(v.own, v.n_own), arr(v.ext, v.n_ext),
                   arr(v.halo, v.n_halo), arr(v.send_offsets, w + 1), arr(v.send_idx, v.n_send),
                   arr(v.recv_offsets, w + 1), arr(v.gather, v.n_ext), arr(v.out_index, v.n_ext))


def make_plan(a: H.CsrMatrix, world: int, rank: int, overlap: int) -> RasPlan:
    """The reference partition (partition_graph + extend_overlap) and this rank's maps (C++, host only)."""
    h = C.c_void_p()
    check(lib.hec_ras_plan_create(a.handle, world, rank, overlap, C.byref(h)))
    try:
        return _plan_from_handle(h)
    finally:
        lib.hec_ras_plan_destroy(h)


@dataclass
class RasReport:
    converged: bool = False
    iterations: int = 0
    final_relative_residual: float = 0.0
    solve_seconds: float = 0.0
    inner_residuals: List[float] = field(default_factory=list)
    allreduces: int = 0
    exchanges: int = 0
    launches: int = 0


class _TorchCallbacks:
    """Host-staged collectives over a torch.distributed group (gloo) for the C++ engine."""

    def __init__(self, plan_view_fn):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self._plan = plan_view_fn
        self.cb_allreduce = L.ALLREDUCE_CB(self._allreduce)
        self.cb_exchange = L.EXCHANGE_CB(self._exchange)

    def _allreduce(self, ctx, buf, count):
        try:
            t = self.torch.from_numpy(np.ctypeslib.as_array(buf, shape=(count,)))
            self.dist.all_reduce(t)
            return 0
        except Exception:  # pragma: no cover - surfaced as HEC_ERUNTIME
            return 1

    def _exchange(self, ctx, send, ns, recv, nr):
        try:
            plan = self._plan()
            s = self.torch.from_numpy(np.ctypeslib.as_array(send, shape=(max(ns, 1),))[:ns].copy())
            r = self.torch.empty(nr, dtype=self.torch.float64)
            self.dist.all_to_all_single(r, s, plan.recv_counts, plan.send_counts)
            if nr:
                np.ctypeslib.as_array(recv, shape=(nr,))[:] = r.numpy()
            return 0
        except Exception:  # pragma: no cover
            return 1


class RasSolver:
    """hec_ras_t: this rank's subdomain of a RAS-preconditioned GMRES (collective calls)."""

    def __init__(self, a: H.CsrMatrix, overlap: int = 1, local: str = "ilu0", fill_level: int = 1,
                 ilut_p: int = 7, ilut_tol: float = 0.1, comm: str = "auto"):
        kind = {"ilu0": 0, "ilut": 1, "iluk": 3}[local]
        spec = L.CommSpec()
        self._callbacks = None
        world, rank, backend = 1, 0, None
        try:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized():
                world, rank, backend = dist.get_world_size(), dist.get_rank(), dist.get_backend()
        except Exception:
            pass
        if comm == "auto":
            comm = "none" if world == 1 else ("nccl" if backend == "nccl" else "callbacks")
        spec.rank, spec.world = rank, world
        if comm == "none":
            spec.kind = L.COMM_NONE
        elif comm == "nccl":
            uid = (C.c_ubyte * 128)()
            if rank == 0:
                check(lib.hec_nccl_unique_id(uid))
            if world > 1:  # rank 0's id to every rank (torch.distributed is the bootstrap channel)
                import torch
                import torch.distributed as dist
                t = torch.tensor(bytearray(uid), dtype=torch.uint8, device="cuda")
                dist.broadcast(t, 0)
                uid = (C.c_ubyte * 128)(*t.cpu().tolist())
            self._uid = uid
            spec.kind = L.COMM_NCCL
            spec.nccl_id = C.cast(self._uid, C.POINTER(C.c_ubyte))
        elif comm == "callbacks":
            self._callbacks = _TorchCallbacks(lambda: self.plan)
            spec.kind = L.COMM_CALLBACKS
            spec.callbacks = L.CommCallbacks(None, self._callbacks.cb_allreduce, self._callbacks.cb_exchange)
        else:
            raise ValueError(f"unknown comm {comm!r}")
        self.comm = comm
        h = C.c_void_p()
        check(lib.hec_ras_create(a.handle, overlap, kind, ilut_p, ilut_tol, fill_level, C.byref(spec), C.byref(h)))
        self._h = h
        ph = C.c_void_p()
        check(lib.hec_ras_get_plan(h, C.byref(ph)))
        self.plan = _plan_from_handle(ph)

    def apply(self, r_own_dev, z_own_dev, stream=None):
        """z = M^-1 r on the owned rows (device tensors); collective."""
        check(lib.hec_ras_apply(self._h, C.c_void_p(H._ptr(r_own_dev)), C.c_void_p(H._ptr(z_own_dev)),
                                C.c_void_p(H._stream(stream)) if stream is not None else None))

    def apply_host(self, r_own) -> np.ndarray:
        rv = H._f64_vec(r_own, self.plan.n_own, "ras apply")
        z = np.empty(self.plan.n_own)
        check(lib.hec_ras_apply_host(self._h, H._p_dbl(rv), H._p_dbl(z)))
        return z

    def gmres(self, b_own, restart: int = 20, max_iters: int = 10000, rel_tol: float = 1e-6,
              abs_tol: float = 0.0):
        """RAS GMRES on the owned rows (host vectors); collective. Returns (x_own, RasReport)."""
        bv = H._f64_vec(b_own, self.plan.n_own, "ras gmres")
        x = np.empty(self.plan.n_own)
        cap = max(max_iters, 0) + 1
        inner = np.empty(cap)
        rep = L.GmresReport()
        cfg = L.GmresConfig(restart, max_iters, rel_tol, abs_tol)
        check(lib.hec_ras_gmres(self._h, H._p_dbl(bv), C.byref(cfg), H._p_dbl(x), C.byref(rep), H._p_dbl(inner),
                                cap))
        ar, ex, la = C.c_longlong(), C.c_longlong(), C.c_longlong()
        check(lib.hec_ras_stats(self._h, C.byref(ar), C.byref(ex), C.byref(la)))
        return x, RasReport(bool(rep.converged), rep.iterations, rep.final_relative_residual, rep.solve_seconds,
                            inner[:min(rep.n_inner, cap)].tolist(), ar.value, ex.value, la.value)

    def gmres_device(self, b_own_dev, x_own_dev, restart: int = 20, max_iters: int = 10000,
                     rel_tol: float = 1e-6, abs_tol: float = 0.0, stream=None) -> RasReport:
        rep = L.GmresReport()
        cfg = L.GmresConfig(restart, max_iters, rel_tol, abs_tol)
        check(lib.hec_ras_gmres_device(self._h, C.c_void_p(H._ptr(b_own_dev)), C.byref(cfg),
                                       C.c_void_p(H._ptr(x_own_dev)), C.byref(rep), None, 0,
                                       C.c_void_p(H._stream(stream)) if stream is not None else None))
        ar, ex, la = C.c_longlong(), C.c_longlong(), C.c_longlong()
        check(lib.hec_ras_stats(self._h, C.byref(ar), C.byref(ex), C.byref(la)))
        return RasReport(bool(rep.converged), rep.iterations, rep.final_relative_residual, rep.solve_seconds, [],
                         ar.value, ex.value, la.value)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:  # (module globals are gone at interpreter exit)
            lib.hec_ras_destroy(self._h)
        self._h = None


class RasGmres:
    """Convenience: RAS-preconditioned GMRES(restart) of a global system, one subdomain per rank."""

    def __init__(self, a: H.CsrMatrix, overlap: int = 1, restart: int = 20, max_iters: int = 10000,
                 rel_tol: float = 1e-6, abs_tol: float = 0.0, local: str = "ilu0", fill_level: int = 1,
                 ilut_p: int = 7, ilut_tol: float = 0.1, device=None, comm: str = "auto"):
        self.solver = RasSolver(a, overlap, local, fill_level, ilut_p, ilut_tol, comm)
        self.plan = self.solver.plan
        self.cfg = dict(restart=restart, max_iters=max_iters, rel_tol=rel_tol, abs_tol=abs_tol)

    def solve(self, b_global):
        """b: global right-hand side (host). Returns (x on the owned rows (host), RasReport)."""
        b_own = np.ascontiguousarray(np.asarray(b_global, dtype=np.float64)[self.plan.own])
        t0 = time.perf_counter()
        x, rep = self.solver.gmres(b_own, **self.cfg)
        rep.solve_seconds = rep.solve_seconds or time.perf_counter() - t0
        return x, rep
