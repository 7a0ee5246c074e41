"""Diagnostics: one RAS GMRES solve on this GPU (world 1) with a capped
iteration count, for ncu launch lists (per-kernel share of an iteration).

    python tools/ras_profile.py [--size 256] [--iters 30]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402
from paper_1606_00541_b200 import ras  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--restart", type=int, default=30)
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s)
    b = H.spmv_csr(a, np.ones(a.n_rows))
    solver = ras.RasSolver(a, overlap=1)
    bd = torch.tensor(b[solver.plan.own], device="cuda")
    xd = torch.empty_like(bd)
    for rep_i in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = solver.gmres_device(bd, xd, restart=args.restart, max_iters=args.iters)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"run {rep_i}: {rep.iterations} iterations, {dt*1e3:.1f} ms, {dt*1e3/max(rep.iterations,1):.3f} ms/iter, "
              f"launches {rep.launches}", flush=True)


if __name__ == "__main__":
    main()
