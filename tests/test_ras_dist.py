"""Multi-GPU RAS layer (paper_1606_00541_b200/ras.py).

CPU (world size 2, gloo): the distributed host logic -- reference partition,
halo plan, all-to-all halo exchange, distributed GMRES -- with the local work
done by the oracle (tests only). Checks: the distributed preconditioner apply
equals the reference's hec::apply with the same blocks bitwise, and GMRES
converges in the reference's iteration count +-1.

GPU: the same driver with the device local work (DeviceOps), world size 1
(NCCL not needed) and world size 2 on one GPU (gloo, host-staged collectives).
"""
import os
import socket

import numpy as np
import pytest

from oracle.oracle import Csr
from util import bits_equal


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleOps:
    """Local subdomain work on the CPU through the oracle (test backend)."""

    def __init__(self, H, a, plan, orc):
        import torch
        self.torch, self.orc, self.plan = torch, orc, plan
        f = H.ilu0(H.csr_submatrix(a, plan.ext))
        self.pl = orc.prepare(Csr.of(f.l))
        self.pu = orc.prepare(Csr.of(f.u), upper=True)
        self.owned = (plan.out_index >= 0).astype(np.int8)
        self.A = Csr(plan.n_own, plan.n_loc, plan.a_rp, plan.a_ci, plan.a_v)

    def vec(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64)

    def apply(self, vloc, z_own):
        x = self.orc.apply(self.plan.n_loc, self.plan.gather, self.owned, self.pl, self.pu, vloc.numpy())
        z_own.copy_(self.torch.from_numpy(x[:self.plan.n_own]))

    def matvec(self, zloc, w_own):
        w_own.copy_(self.torch.from_numpy(self.orc.spmv(self.A, zloc.numpy())))

    def mgs(self, w, v_prev, h_prev, v_next, out):
        if v_prev is not None:
            w.sub_(h_prev * v_prev)
        out.copy_(self.torch.dot(w, v_next).reshape(1))

    def scale(self, y, x, s):
        y.copy_(x / s)

    def combine(self, j, xc, V, ldv, y):
        n = self.plan.n_own
        acc = self.torch.zeros(n, dtype=self.torch.float64)
        for i in range(j):
            acc = acc + y[i] * V[i * ldv:i * ldv + n]
        xc.copy_(acc)

    def add(self, x, d):
        x.add_(d)

    def sqrt(self, a, out):
        out.copy_(self.torch.sqrt(a))

    def to_host(self, t):
        return t.numpy().copy()

    def from_host(self, arr):
        return self.torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64))

    def copy(self, dst, src):
        dst.copy_(src)

    def residual(self, r, b, ax):
        self.torch.sub(b, ax, out=r)

    def sub(self, V, i, ldv, n):
        return V[i * ldv:i * ldv + n]


def _gloo_worker(rank, world, port, dims, restart, queue):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1606_00541_b200 as H
        from paper_1606_00541_b200 import ras
        from oracle import load_oracle, load_reference
        orc, ref = load_oracle(), load_reference()
        a = H.gen_poisson7(*dims)
        plan = ras.make_plan(a, world, rank, 1)
        ops = OracleOps(H, a, plan, orc)
        comm = ras.TorchComm(plan, torch.device("cpu"))
        # 1) distributed apply == reference hec::apply with `world` RAS blocks, bitwise
        r = np.random.default_rng(7).uniform(-1, 1, a.n_rows)
        vloc = torch.zeros(plan.n_loc, dtype=torch.float64)
        vloc[:plan.n_own] = torch.from_numpy(r[plan.own])
        comm.exchange(vloc)
        z = torch.zeros(plan.n_own, dtype=torch.float64)
        ops.apply(vloc, z)
        A = Csr.of(a)
        want = ref.apply(ref.precond(A, "ras", world, 1), r)
        apply_ok = bits_equal(z.numpy(), want[plan.own])
        # 2) distributed GMRES vs the reference's RAS GMRES
        b = ref.spmv(A, np.ones(a.n_rows))
        x, rep = ras.gmres(ops, comm, plan, b[plan.own], restart=restart)
        xs = [None] * world
        dist.all_gather_object(xs, (plan.own, x.numpy()))
        _, rrep = ref.gmres(A, b, ref.precond(A, "ras", world, 1), restart=restart)
        if rank == 0:
            xg = np.zeros(a.n_rows)
            for own, xv in xs:
                xg[own] = xv
            res = np.linalg.norm(b - ref.spmv(A, xg)) / np.linalg.norm(b)
            queue.put(dict(apply_ok=apply_ok, iters=rep.iterations, ref_iters=rrep["iterations"],
                           conv=rep.converged, rel=rep.final_relative_residual, true_rel=res,
                           allreduces=rep.allreduces, exchanges=rep.exchanges))
        else:
            queue.put(dict(apply_ok=apply_ok))
    finally:
        dist.destroy_process_group()


def test_plan_invariants(H):
    from paper_1606_00541_b200 import ras
    a = H.gen_poisson7(9, 8, 7)
    for world in (1, 2, 3, 5):
        plans = [ras.make_plan(a, world, r, 1) for r in range(world)]
        own_all = np.concatenate([p.own for p in plans])
        assert np.array_equal(np.sort(own_all), np.arange(a.n_rows))      # every row owned exactly once
        for p in plans:
            assert not np.intersect1d(p.own, p.halo).size
            assert np.all(p.gather < p.n_loc) and np.all(p.gather >= 0)
            owned = p.out_index >= 0
            assert np.array_equal(np.sort(p.ext[owned]), p.own)           # restriction = own rows
            assert np.array_equal(p.gather[owned], p.out_index[owned])
            for q in range(world):                                         # send / receive sizes match
                assert len(plans[q].send_idx[p.rank]) == p.recv_counts[q]


@pytest.mark.parametrize("world", [2, 3])
def test_ras_gmres_gloo_cpu(ref, world):
    torch = pytest.importorskip("torch")
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, (10, 9, 8), 20, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o["apply_ok"] for o in out), "distributed apply differs from the reference's hec::apply"
    main = next(o for o in out if "iters" in o)
    assert main["conv"] and main["rel"] <= 1e-6 and main["true_rel"] <= 1e-6
    assert abs(main["iters"] - main["ref_iters"]) <= 1, main
    assert main["exchanges"] > 0 and main["allreduces"] > 0


def _gpu_worker(rank, world, port, queue):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1606_00541_b200 as H
        from paper_1606_00541_b200 import ras
        from oracle import load_reference
        ref = load_reference()
        a = H.gen_poisson7(16, 15, 14)
        A = Csr.of(a)
        b = ref.spmv(A, np.ones(a.n_rows))
        solver = ras.RasGmres(a, overlap=1, restart=30)
        x, rep = solver.solve(b)
        xs = [None] * world
        dist.all_gather_object(xs, (solver.plan.own, x.cpu().numpy()))
        _, rrep = ref.gmres(A, b, ref.precond(A, "ras", world, 1), restart=30)
        if rank == 0:
            xg = np.zeros(a.n_rows)
            for own, xv in xs:
                xg[own] = xv
            queue.put(dict(iters=rep.iterations, ref_iters=rrep["iterations"], conv=rep.converged,
                           true_rel=float(np.linalg.norm(b - ref.spmv(A, xg)) / np.linalg.norm(b))))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ras_gmres_device_world1(H, ref):
    torch = pytest.importorskip("torch")
    from paper_1606_00541_b200 import ras
    a = H.gen_poisson7(20, 18, 16)
    A = Csr.of(a)
    b = ref.spmv(A, np.ones(a.n_rows))
    solver = ras.RasGmres(a, overlap=1, restart=30)
    x, rep = solver.solve(b)
    _, rrep = ref.gmres(A, b, ref.precond(A, "ras", 1, 1), restart=30)
    assert rep.converged and abs(rep.iterations - rrep["iterations"]) <= 1, (rep.iterations, rrep)
    xr = x.cpu().numpy()
    assert np.linalg.norm(b - ref.spmv(A, xr)) / np.linalg.norm(b) <= 1e-6
    # the device apply on one block is the reference apply bitwise
    r = np.random.default_rng(3).uniform(-1, 1, a.n_rows)
    vloc = torch.tensor(r, device="cuda")
    z = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
    solver.ops.apply(vloc, z)
    torch.cuda.synchronize()
    assert bits_equal(z.cpu().numpy(), ref.apply(ref.precond(A, "ras", 1, 1), r))


@pytest.mark.gpu
def test_ras_gmres_device_world2_one_gpu(ref):
    torch = pytest.importorskip("torch")
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out["conv"] and out["true_rel"] <= 1e-6
    assert abs(out["iters"] - out["ref_iters"]) <= 1, out
