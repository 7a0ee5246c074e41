"""RAS-preconditioned GMRES time-to-solution, one subdomain per GPU.

    python tools/ras_bench.py --size 64                      # 1 GPU
    torchrun --nproc-per-node G tools/ras_bench.py --size 256
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=64)
    ap.add_argument("--restart", type=int, default=30)
    ap.add_argument("--overlap", type=int, default=1)
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--max-iters", type=int, default=10000)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_1606_00541_b200 as H
    from paper_1606_00541_b200 import ras
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    if world > 1:
        dist.init_process_group(args.backend)
    s = args.size
    t0 = time.time()
    a = H.gen_poisson7(s, s, s)
    b = H.spmv_csr(a, np.ones(a.n_rows), workers=os.cpu_count())
    solver = ras.RasGmres(a, overlap=args.overlap, restart=args.restart, max_iters=args.max_iters)
    t_setup = time.time() - t0
    solver.solve(b)  # warm-up (device layouts, workspaces)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t1 = time.perf_counter()
    x, rep = solver.solve(b)
    torch.cuda.synchronize()
    t = time.perf_counter() - t1
    if world > 1:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    err = float((x - 1.0).abs().max().item())
    if world > 1:
        e = torch.tensor([err], dtype=torch.float64, device="cuda")
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
        err = float(e.item())
    if rank == 0:
        print(json.dumps(dict(size=s, world=world, iterations=rep.iterations, converged=rep.converged,
                              rel=rep.final_relative_residual, seconds=round(t, 4),
                              ms_per_iter=round(1e3 * t / max(rep.iterations, 1), 3), max_err=err,
                              allreduces=rep.allreduces, exchanges=rep.exchanges, setup_s=round(t_setup, 1),
                              n_own=solver.plan.n_own, halo=len(solver.plan.halo))), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
