"""SM-cycle breakdown of one chunk for solver warp 5 (traced kernel, words 56..63),
on the synthetic `chains` pattern of tools/wavebench.py (diagnostics).

python tools/stamps.py --S 64 512 --C 1
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1606_00541_b200 as H  # noqa: E402
from wavebench import build  # noqa: E402

NAMES = ["bar_full", "header", "deps", "dd", "xv", "stored", "x", "published"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, nargs="*", default=[64, 512])
    ap.add_argument("--C", type=int, default=1)
    ap.add_argument("--D", type=int, default=400)
    ap.add_argument("--kind", default="chains")
    args = ap.parse_args()
    import torch
    for S in args.S:
        p = H.prepare_lower(build(args.kind, S, args.D, args.C))
        t = H.DeviceTri.create(p, strategy=2, ctas=args.C)
        b = torch.ones(p.n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(b)
        for _ in range(2):
            t.solve(b, x)
        tr, c0 = t.solve_traced(b, x)
        tr = tr.astype(np.int64)
        nw = t.info()["threads"] // 32 - 4
        ws = 5 if nw > 5 else 0  # the traced kernel stamps warp 5 (or warp 0)
        cyc = tr[:, 56:64] if ws == 5 else tr[:, 48:56]
        ok = cyc[:, 7] > 0
        if not ok.any():
            print(f"S={S}: no stamps (solver warp 5 absent: {t.info()['threads'] // 32 - 4} solver warps)")
            continue
        med = np.median(cyc[ok], axis=0)
        done = tr[:, 10 + 3 * ws]
        per = np.diff(done[c0[0]:c0[1]])
        print(f"S={S} C={args.C} warps={nw}: chunk period p50 {np.median(per):.0f} ns; warp {ws} cycles from loop top: "
              + "  ".join(f"{n} {int(v)}" for n, v in zip(NAMES, med)), flush=True)


if __name__ == "__main__":
    main()
