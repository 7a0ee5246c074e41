"""Run a few solves of one configuration (target for ncu captures).

python tools/one_solve.py --stencil 7 --size 128 --which L --reps 3 [--strategy 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stencil", default="7")
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--which", default="L")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--strategy", type=int, default=2)
    ap.add_argument("--ctas", type=int, default=0)
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s) if args.stencil == "7" else H.gen_poisson27(s, s, s)
    f = H.ilu0(a)
    p = H.prepare_lower(f.l) if args.which == "L" else H.prepare_upper(f.u)
    t = H.DeviceTri.create(p, strategy=args.strategy, ctas=args.ctas)
    b = torch.ones(a.n_rows, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(args.reps):
        t.solve(b, x)
    torch.cuda.synchronize()
    print(t.info())


if __name__ == "__main__":
    main()
