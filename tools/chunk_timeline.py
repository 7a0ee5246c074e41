"""Per-chunk timeline of one CTA from the traced kernel (diagnostics):
issue -> landed (waiter) -> group sees blob -> released -> done, in ns.

python tools/chunk_timeline.py --chains 32 --C 1 [--first 200 --count 12]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1606_00541_b200 as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stencil", default="7")
    ap.add_argument("--size", type=int, default=0)
    ap.add_argument("--chains", type=int, default=32)
    ap.add_argument("--C", type=int, default=1)
    ap.add_argument("--D", type=int, default=2000)
    ap.add_argument("--cta", type=int, default=-1)
    ap.add_argument("--extra", type=int, default=0)
    ap.add_argument("--first", type=int, default=200)
    ap.add_argument("--count", type=int, default=12)
    args = ap.parse_args()
    import torch
    if args.size:
        s = args.size
        a = H.gen_poisson7(s, s, s) if args.stencil == "7" else H.gen_poisson27(s, s, s)
        L = H.ilu0(a).l
    else:
        from wavebench import build
        L = build("chains", args.chains, args.D, args.C, args.extra)
    p = H.prepare_lower(L)
    t = H.DeviceTri.create(p, strategy=2, ctas=args.C if not args.size else 0)
    b = torch.ones(p.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(2):
        t.solve(b, x)
    tr, c0 = t.solve_traced(b, x)
    tr = tr.astype(np.int64)
    info = t.info()
    nw = info["group"] * info["groups"]  # solver warps (role warps vary with the shape)
    T = np.where(tr > 0, tr - tr[:, 0].min(), -1)
    c = args.cta if args.cta >= 0 else (len(c0) - 1) // 2
    lo, hi = c0[c], c0[c + 1]
    sees = T[:, 8:8 + 3 * nw:3]
    rel = T[:, 9:9 + 3 * nw:3]
    done = T[:, 10:10 + 3 * nw:3]
    m = lambda a: np.where(a >= 0, a, np.iinfo(np.int64).max).min(axis=1)
    S, Rl, D = m(sees), m(rel), done.max(axis=1)
    print(f"{info['ctas']} CTAs, {nw} solver warps, CTA {c}: chunks {hi - lo}")
    issue = T[lo:hi, 0]
    print("issue period p50 %.0f ns; landed-issue p50 %.0f; release-landed p50 %.0f; done-release p50 %.0f; "
          "period(done) p50 %.0f" % (np.median(np.diff(issue)), np.median(T[lo:hi, 1] - issue),
                                    np.median(Rl[lo:hi] - T[lo:hi, 1]), np.median(D[lo:hi] - Rl[lo:hi]),
                                    np.median(np.diff(D[lo:hi]))))
    print(" j    p.top  p.slot   issue  p.issued  landed    ready     sees  release     done")
    for j in range(lo + args.first, min(hi, lo + args.first + args.count)):
        print(f"{j-lo:4d} {T[j,4]:8d} {T[j,5]:8d} {T[j,0]:8d} {T[j,6]:8d} {T[j,1]:8d} {T[j,3]:8d} {S[j]:8d} "
              f"{Rl[j]:8d} {D[j]:8d}")


if __name__ == "__main__":
    main()
