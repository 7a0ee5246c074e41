"""Per-rank local work of a G-way RAS on one GPU (diagnostics): for rank r of
world G, the local ILU apply and SpMV of its block (as hec_ras_create builds
them), timed alone -- what one GPU of a G-GPU run spends per GMRES iteration
outside communication and Gram-Schmidt.

    python tools/ras_rank_local.py --size 256 --world 8 [--ranks 0 3 7]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402
from paper_1606_00541_b200 import ras  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--ranks", type=int, nargs="*", default=None)
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s)
    for r in (args.ranks if args.ranks else range(args.world)):
        plan = ras.make_plan(a, args.world, r, 1)
        f = H.ilu0(H.csr_submatrix(a, plan.ext))
        pl, pu = H.prepare_lower(f.l), H.prepare_upper(f.u)
        dp = H.DevicePrecond.create_local(plan.n_loc, plan.n_own, pl, pu, plan.gather, plan.out_index)
        li, ui = dp.info()
        rows = [0] + [0] * plan.n_own
        A = H.csr_submatrix(a, plan.own)  # timing only: same nnz pattern per row as the local SpMV
        sp = H.DeviceSpmv(A)
        v = torch.rand(plan.n_loc, dtype=torch.float64, device="cuda")
        z = torch.empty(plan.n_own, dtype=torch.float64, device="cuda")
        xa = torch.rand(A.n_cols, dtype=torch.float64, device="cuda")
        w = torch.empty(A.n_rows, dtype=torch.float64, device="cuda")
        for _ in range(3):
            dp.apply(v, z)
            sp.run(xa, w)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        for _ in range(10):
            dp.apply(v, z)
        e[1].record()
        for _ in range(10):
            sp.run(xa, w)
        e[2].record()
        torch.cuda.synchronize()
        print(f"world {args.world} rank {r}: own {plan.n_own} halo {len(plan.halo)} block {len(plan.ext)} "
              f"nlev L/U {pl.schedule.nlev}/{pu.schedule.nlev} layout L/U {li['layout']}/{ui['layout']} "
              f"apply {e[0].elapsed_time(e[1]) / 10:.3f} ms  spmv {e[1].elapsed_time(e[2]) / 10:.3f} ms", flush=True)
        del rows


if __name__ == "__main__":
    main()
