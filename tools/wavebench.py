"""Synthetic lower-triangular patterns that isolate the wave kernel's costs
(diagnostics; run on the GPU box).

  chains   C independent blocks; in each, column s (of S) is a chain of D rows
           (row (s,k) depends on (s,k-1)); warp-local dependencies only.
           time / D = per-level cost inside a CTA.
  warps    as chains, plus (s,k) <- (s-1,k-1): cross-warp handoffs inside a CTA.
  ctas     one S*C x D grid, (s,k) <- (s,k-1), (s-1,k-1): the dependency chain
           crosses every CTA boundary once per level shift (slab-like).

python tools/wavebench.py --S 512 --D 400 --C 148
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def build(kind, S, D, C, extra=0):
    # index of (block, s, k) = block*S*D + s*D + k  (column-major chains)
    rows, cols, vals = [], [], []
    nb = C if kind in ("chains", "warps") else 1
    SS = S if kind in ("chains", "warps") else S * C
    n = nb * SS * D
    idx = np.arange(n, dtype=np.int64).reshape(nb, SS, D)
    # diagonal
    rows.append(idx.ravel()); cols.append(idx.ravel()); vals.append(np.full(n, 4.0))
    # (s,k) <- (s,k-1)
    rows.append(idx[:, :, 1:].ravel()); cols.append(idx[:, :, :-1].ravel()); vals.append(np.full(nb * SS * (D - 1), -1.0))
    for e in range(1, min(extra, SS - 1) + 1):  # wider rows: (s, k) <- (s - e, k - 1)
        dst, src = idx[:, e:, 1:], idx[:, :-e, :-1]
        rows.append(dst.ravel()); cols.append(src.ravel()); vals.append(np.full(dst.size, -0.01))
    if kind in ("warps", "ctas"):
        rows.append(idx[:, 1:, 1:].ravel()); cols.append(idx[:, :-1, :-1].ravel())
        vals.append(np.full(nb * (SS - 1) * (D - 1), -0.5))
    r = np.concatenate(rows); c = np.concatenate(cols); v = np.concatenate(vals)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rp = np.zeros(n + 1, dtype=np.int32)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    return H.CsrMatrix.from_arrays(n, n, rp, c.astype(np.int32), v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=int, default=512)
    ap.add_argument("--D", type=int, default=400)
    ap.add_argument("--C", type=int, default=148)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--kinds", nargs="*", default=["chains", "warps", "ctas"])
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--extra", type=int, default=0, help="extra dependencies per row (row width 1 + extra)")
    args = ap.parse_args()
    import torch
    for kind in args.kinds:
        t0 = time.time()
        L = build(kind, args.S, args.D, args.C, args.extra)
        p = H.prepare_lower(L)
        t = H.DeviceTri.create(p, strategy=2, ctas=args.C, threads=args.threads)
        info = t.info()
        b = torch.ones(p.n, dtype=torch.float64, device="cuda")
        x = torch.empty_like(b)
        for _ in range(2):
            t.solve(b, x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(args.reps):
            e0.record()
            t.solve(b, x)
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        m = float(np.median(ms))
        nl = p.schedule.nlev
        print(f"{kind:7s} n={p.n} nlev={nl} chunks={info['chunks']} ctas={info['ctas']}  {m*1e3:.1f} us  "
              f"{m*1e6/nl:.1f} ns/level  (setup {time.time()-t0:.1f}s)", flush=True)
        if args.trace:
            tr, c0 = t.solve_traced(b, x)
            tr = tr.astype(np.int64)
            nw = info["group"] * info["groups"]  # solver warps
            T = np.where(tr > 0, tr - tr[:, 0].min(), -1)
            rs, dd, dn = T[:, 8:8 + 3 * nw:3], T[:, 9:9 + 3 * nw:3], T[:, 10:10 + 3 * nw:3]
            pct = lambda a: "p10 %.0f p50 %.0f p90 %.0f" % tuple(np.percentile(a, [10, 50, 90]))
            print("   TMA issue -> waiter sees:", pct(T[:, 1] - T[:, 0]))
            print("   waiter sees -> ready:    ", pct(T[:, 3] - T[:, 1]))
            print("   ready -> first warp sees:", pct(rs.min(1) - T[:, 3]))
            print("   warp work (deps->done):  ", pct((dn - dd)[dd >= 0]))
            print("   warp seen->deps:         ", pct((dd - rs)[dd >= 0]))
            c = 5
            lo = c0[c]
            for j in range(lo + 50, lo + 56):
                print(f"   j={j-lo} issue {T[j,0]} sees {T[j,1]} ready {T[j,3]} | "
                      + " ".join(f"{rs[j,w]}/{dd[j,w]}/{dn[j,w]}" for w in (0, 5, 10, 15)))


if __name__ == "__main__":
    main()
