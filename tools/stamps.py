"""SM-clock stamps of solver warp 0 after its dependency wait (traced kernel,
words 48..53) and the chunk period (diagnostics).

python tools/stamps.py --stencil 7 --size 256      (or --chains S --C C)
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1606_00541_b200 as H  # noqa: E402

NAMES = ["(0)", "gathers", "fp", "stores", "arrive", "x stored"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stencil", default="7")
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--chains", type=int, default=0)
    ap.add_argument("--C", type=int, default=148)
    ap.add_argument("--D", type=int, default=400)
    args = ap.parse_args()
    import torch
    if args.chains:
        from wavebench import build
        L = build("chains", args.chains, args.D, args.C)
    else:
        s = args.size
        a = H.gen_poisson7(s, s, s) if args.stencil == "7" else H.gen_poisson27(s, s, s)
        L = H.ilu0(a).l
    p = H.prepare_lower(L)
    t = H.DeviceTri.create(p, strategy=2, ctas=args.C)
    b = torch.ones(p.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(2):
        t.solve(b, x)
    tr, c0 = t.solve_traced(b, x)
    tr = tr.astype(np.int64)
    info = t.info()
    cyc = tr[:, 48:54]
    ok = cyc[:, 5] > 0
    med = np.median(cyc[ok], axis=0)
    T = np.where(tr > 0, tr - tr[:, 0].min(), -1)
    nw = info["group"] * info["groups"]  # solver warps (role warps vary with the shape)
    dd, dn = T[:, 9:9 + 3 * nw:3], T[:, 10:10 + 3 * nw:3]
    last = dn.max(axis=1)
    cm = (len(c0) - 1) // 2
    per = np.diff(last[c0[cm]:c0[cm + 1]])
    # handoff: chunk j released (deps) vs chunk j-1 done (max over its warps)
    dmin = np.where(dd >= 0, dd, np.iinfo(np.int64).max).min(axis=1)
    lo, hi = c0[cm], c0[cm + 1]
    hand = dmin[lo + 1:hi] - last[lo:hi - 1]
    print(f"{info['ctas']} CTAs x {nw} solver warps, chunks {info['chunks']}; CTA {cm}: period p50 {np.median(per):.0f} ns, "
          f"release(j) - done(j-1) p50 {np.median(hand):.0f} ns; warp 0 cycles after its wait: "
          + "  ".join(f"{n} {int(v)}" for n, v in zip(NAMES[1:], med[1:])), flush=True)


if __name__ == "__main__":
    main()
