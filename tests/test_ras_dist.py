"""Multi-GPU RAS layer: the C++ plan (csrc/host/ras_plan.cpp), the device
engine (csrc/cuda/gmres_engine.cu, comm.cpp) and its Python face (ras.py).

CPU (gloo, world sizes 2 and 3): the product's C++ plan with the local work done
by the oracle and the CGS2 GMRES restated in tests/ras_model.py. Checks: the
distributed preconditioner apply equals the reference's hec::apply with the same
blocks bitwise; GMRES converges in the reference's iteration count +-1.

GPU: the C++ engine through the C-ABI (hec_ras_create / apply / gmres): world
size 1, and world size 2 on one GPU (two processes, host-callback collectives
over gloo) -- the apply bitwise equal to the reference's rows, GMRES iterations
within +-1. (NCCL runs in the driver's multi-GPU bench, one process per GPU.)
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


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _gather_global(plan, x, n):
    import torch.distributed as dist
    xs = [None] * plan.world
    dist.all_gather_object(xs, (plan.own, np.asarray(x)))
    xg = np.zeros(n)
    for own, xv in xs:
        xg[own] = xv
    return xg


def _gloo_worker(rank, world, port, dims, restart, queue):
    import torch.distributed as dist
    _init(rank, world, port)
    try:
        import paper_1606_00541_b200 as H
        from paper_1606_00541_b200 import ras
        from oracle import load_oracle, load_reference
        import ras_model
        orc, ref = load_oracle(), load_reference()
        a = H.gen_poisson7(*dims)
        plan = ras.make_plan(a, world, rank, 1)
        local = ras_model.OracleLocal(H, a, plan, orc)
        comm = ras_model.GlooComm(plan)
        # 1) distributed apply == reference hec::apply with `world` RAS blocks, bitwise
        r = np.random.default_rng(7).uniform(-1, 1, a.n_rows)
        vloc = np.zeros(plan.n_loc)
        vloc[:plan.n_own] = r[plan.own]
        comm.exchange(vloc)
        z = local.apply(vloc)
        A = Csr.of(a)
        want = ref.apply(ref.precond(A, "ras", world, 1), r)
        apply_ok = bits_equal(z, want[plan.own])
        # 2) distributed GMRES (the engine's algorithm) vs the reference's RAS GMRES
        b = ref.spmv(A, np.ones(a.n_rows))
        x, rep = ras_model.gmres(local, comm, plan, b[plan.own], restart=restart)
        xg = _gather_global(plan, x, a.n_rows)
        _, rrep = ref.gmres(A, b, ref.precond(A, "ras", world, 1), restart=restart)
        if rank == 0:
            res = np.linalg.norm(b - ref.spmv(A, xg)) / np.linalg.norm(b)
            queue.put(dict(apply_ok=apply_ok, iters=rep["iterations"], ref_iters=rrep["iterations"],
                           conv=rep["converged"], rel=rep["rel"], true_rel=res, allreduces=rep["allreduces"],
                           exchanges=rep["exchanges"]))
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
            assert np.array_equal(p.part_of[p.halo], np.sort(p.part_of[p.halo]))  # halo by owner
            for q in range(world):                                         # send / receive sizes match
                assert plans[q].send_counts[p.rank] == p.recv_counts[q]
                seg = p.halo[p.recv_offsets[q]:p.recv_offsets[q + 1]]
                assert np.array_equal(plans[q].own[plans[q].send_idx[plans[q].send_offsets[p.rank]:
                                                                       plans[q].send_offsets[p.rank + 1]]], seg)


def test_plan_matches_reference_partition(H, ref):
    # own = the reference's part, ext = the reference's extended part (precond.cpp:74-96)
    from paper_1606_00541_b200 import ras
    a = H.gen_poisson7(10, 9, 8)
    A = Csr.of(a)
    for world in (2, 4):
        bag = ref.precond(A, "ras", world, 1)
        part_of, offs, ext_rows = bag.ints("part_of"), bag.ints("offsets"), bag.ints("ext_rows")
        for r in range(world):
            p = ras.make_plan(a, world, r, 1)
            assert np.array_equal(p.part_of, part_of)
            assert np.array_equal(p.own, np.flatnonzero(part_of == r))
            assert np.array_equal(p.ext, ext_rows[offs[r]:offs[r + 1]])


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


def _check_device_ras(H, ref, world, rank, dims, queue):
    import torch
    from paper_1606_00541_b200 import ras
    a = H.gen_poisson7(*dims)
    A = Csr.of(a)
    b = ref.spmv(A, np.ones(a.n_rows))
    solver = ras.RasSolver(a, overlap=1)
    plan = solver.plan
    # the distributed apply: rank's rows of the reference's apply(ras, world blocks), bitwise
    r = np.random.default_rng(3).uniform(-1, 1, a.n_rows)
    z = solver.apply_host(r[plan.own])
    want = ref.apply(ref.precond(A, "ras", world, 1), r)
    apply_ok = bits_equal(z, want[plan.own])
    rd = torch.tensor(r[plan.own], device="cuda")
    zd = torch.empty_like(rd)
    solver.apply(rd, zd)
    torch.cuda.synchronize()
    apply_dev_ok = bits_equal(zd.cpu().numpy(), want[plan.own])
    x, rep = solver.gmres(b[plan.own], restart=30)
    xg = _gather_global(plan, x, a.n_rows) if world > 1 else x
    _, rrep = ref.gmres(A, b, ref.precond(A, "ras", world, 1), restart=30)
    out = dict(apply_ok=apply_ok and apply_dev_ok, iters=rep.iterations, ref_iters=rrep["iterations"],
               conv=rep.converged, allreduces=rep.allreduces, exchanges=rep.exchanges,
               true_rel=float(np.linalg.norm(b - ref.spmv(A, xg)) / np.linalg.norm(b)), comm=solver.comm)
    if queue is not None:
        queue.put(out)
    return out


def _gpu_worker(rank, world, port, dims, queue):
    import torch
    import torch.distributed as dist
    _init(rank, world, port)
    try:
        torch.cuda.set_device(0)
        import paper_1606_00541_b200 as H
        from oracle import load_reference
        _check_device_ras(H, load_reference(), world, rank, dims, queue)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ras_device_world1(H, ref):
    out = _check_device_ras(H, ref, 1, 0, (20, 18, 16), None)
    assert out["apply_ok"], "RAS apply differs from the reference"
    assert out["conv"] and out["true_rel"] <= 1e-6
    assert abs(out["iters"] - out["ref_iters"]) <= 1, out
    assert out["comm"] == "none" and out["allreduces"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_ras_device_multi_rank_one_gpu(ref, world):
    torch = pytest.importorskip("torch")
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, (16, 15, 14), q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for o in outs:
        assert o["apply_ok"], "distributed RAS apply differs from the reference's rows"
        assert o["conv"] and o["true_rel"] <= 1e-6
        assert abs(o["iters"] - o["ref_iters"]) <= 1, o
        assert o["comm"] == "callbacks" and o["exchanges"] > 0
        # two all-reduces per iteration plus one per norm (CGS2), not j + 2
        assert o["allreduces"] <= 2 * o["iters"] + 2 * (o["iters"] // 30 + 2)


@pytest.mark.gpu
def test_ras_nccl_backend_one_rank(H, ref):
    # the NCCL backend end to end on one rank: libnccl opened at run time (sharing the
    # copy torch loaded), a one-rank communicator, every all-reduce of the engine through
    # ncclAllReduce on the solve's stream; same iterations and apply as without comm
    pytest.importorskip("torch")
    from paper_1606_00541_b200 import _lib, ras
    assert _lib.lib.hec_nccl_version() > 0
    a = H.gen_poisson7(20, 18, 16)
    A = Csr.of(a)
    b = ref.spmv(A, np.ones(a.n_rows))
    s1, s0 = ras.RasSolver(a, overlap=1, comm="nccl"), ras.RasSolver(a, overlap=1, comm="none")
    x1, r1 = s1.gmres(b, restart=30)
    x0, r0 = s0.gmres(b, restart=30)
    assert r1.converged and r1.iterations == r0.iterations and r1.allreduces > 0 and r0.allreduces == 0
    assert bits_equal(x1, x0)  # a one-rank sum changes nothing
    r = np.random.default_rng(5).uniform(-1, 1, a.n_rows)
    assert bits_equal(s1.apply_host(r), s0.apply_host(r))
