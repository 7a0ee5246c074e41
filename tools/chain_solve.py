"""Run the wave solve a few times on a synthetic pattern of tools/wavebench.py
(target for ncu source-level captures; diagnostics).

ncu --set full --import-source on -k regex:k_wave -s 2 -c 1 python tools/chain_solve.py --S 64 --C 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1606_00541_b200 as H  # noqa: E402
from wavebench import build  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=64)
    ap.add_argument("--C", type=int, default=1)
    ap.add_argument("--D", type=int, default=2000)
    ap.add_argument("--kind", default="chains")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--extra", type=int, default=0)
    args = ap.parse_args()
    import torch
    p = H.prepare_lower(build(args.kind, args.S, args.D, args.C, args.extra))
    t = H.DeviceTri.create(p, strategy=2, ctas=args.C)
    b = torch.ones(p.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(args.reps):
        t.solve(b, x)
    torch.cuda.synchronize()
    print(t.info())


if __name__ == "__main__":
    main()
