"""A/B of ILU-apply variants on one box: prints ms per apply of the current build
for the configs given (env knobs are read at DevicePrecond construction).

    HEC_APPLY_SCATTER=1 python tools/apply_ab.py --size 256
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stencil", default="7")
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s) if args.stencil == "7" else H.gen_poisson27(s, s, s)
    f = H.ilu0(a)
    pl, pu = H.prepare_lower(f.l), H.prepare_upper(f.u)
    dp = H.DevicePrecond.create(a.n_rows, pl, pu)
    info = dp.info() if hasattr(dp, "info") else None
    b = torch.rand(a.n_rows, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(3):
        dp.apply(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        dp.apply(b, x)
    e1.record()
    torch.cuda.synchronize()
    print(f"{args.stencil}-pt {s}^3 env={ {k: v for k, v in os.environ.items() if k.startswith('HEC_')} }: "
          f"{e0.elapsed_time(e1) / args.reps:.4f} ms per apply, ctas={info[0]['ctas'] if info else '?'}", flush=True)


if __name__ == "__main__":
    main()
