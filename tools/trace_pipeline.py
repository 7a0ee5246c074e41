"""Timeline of one PIPELINE solve (diagnostics; run on the GPU box).

python tools/trace_pipeline.py --stencil 7 --size 128 --ctas 148
Prints, per event pair, the distribution over chunks, the per-CTA busy/idle
split and the longest cross-CTA handoff chains.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def q(a):
    a = np.asarray(a, dtype=np.float64)
    if a.size == 0:
        return "n/a"
    return "p10 %.0f  p50 %.0f  p90 %.0f  mean %.0f  max %.0f" % (
        np.percentile(a, 10), np.percentile(a, 50), np.percentile(a, 90), a.mean(), a.max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stencil", default="7")
    ap.add_argument("--size", type=int, default=128)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--upper", action="store_true")
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s) if args.stencil == "7" else H.gen_poisson27(s, s, s)
    f = H.ilu0(a)
    p = H.prepare_upper(f.u) if args.upper else H.prepare_lower(f.l)
    t = H.DeviceTri.create(p, strategy=2, ctas=args.ctas, threads=args.threads)
    info = t.info()
    print(info)
    b = torch.ones(a.n_rows, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(3):
        t.solve(b, x)
    torch.cuda.synchronize()
    tr, c0 = t.solve_traced(b, x)
    tr = tr.astype(np.int64)
    nw = info["group"] * info["groups"]  # solver warps (role warps vary with the shape)
    t0 = tr[:, 0].min()
    T = np.where(tr > 0, tr - t0, -1)
    rs = T[:, 8:8 + 3 * nw:3]     # ready seen per warp
    dd = T[:, 9:9 + 3 * nw:3]     # deps satisfied (only for non-empty segments)
    dn = T[:, 10:10 + 3 * nw:3]   # done per warp
    last = dn.max(axis=1)
    print(f"chunks {len(T)}  span {last.max()/1e3:.1f} us  solver warps {nw}")
    print("blob issue -> waiter sees blob (ns): ", q(T[:, 1] - T[:, 0]))
    print("waiter: blob -> halo staged:         ", q(T[:, 2] - T[:, 1]))
    print("waiter: halo -> ready:               ", q(T[:, 3] - T[:, 2]))
    busy = dd >= 0
    print("ready -> warp sees ready:            ", q((rs - T[:, 3:4])[busy]))
    print("warp sees ready -> deps satisfied:   ", q((dd - rs)[busy]))
    print("deps satisfied -> warp done:         ", q((dn - dd)[busy]))
    print("first warp ready-seen -> last done:  ", q(last - rs.min(axis=1)))
    # (SM-clock stamps of solver warp 0: tools/stamps.py)
    # per warp: how long after the previous chunk's done does it see ready
    for c in [0, 1, 70, len(c0) - 2]:
        lo, hi = c0[c], c0[c + 1]
        if hi - lo < 3:
            continue
        per = np.diff(last[lo:hi])
        print(f"CTA {c}: chunks {hi-lo} first {rs[lo].min()/1e3:.1f} us last {last[hi-1]/1e3:.1f} us "
              f"period p50 {np.median(per):.0f} ns mean {per.mean():.0f} ns")
        # warp-level gaps: for each warp, idle time between done(j-1) and deps-satisfied(j)
        for w in range(nw):
            m = busy[lo:hi, w]
            if m.sum() < 3:
                continue
            wait_ready = (rs[lo + 1:hi, w] - dn[lo:hi - 1, w])
            wait_deps = (dd[lo:hi, w] - rs[lo:hi, w])[m]
            work = (dn[lo:hi, w] - dd[lo:hi, w])[m]
            print(f"   warp {w:2d} busy chunks {m.sum():4d}  wait-ready p50 {np.median(wait_ready):6.0f}  "
                  f"wait-deps p50 {np.median(wait_deps):6.0f}  work p50 {np.median(work):6.0f}  ns")
    # raw timeline of a few consecutive chunks (ns, relative to the first issue)
    for c in [0, 70]:
        lo = c0[c]
        print(f"CTA {c} chunks 200..205: issue / waiter-sees / halo / ready ; per warp ready-seen,deps,done (-1 = empty)")
        for j in range(lo + 200, min(lo + 206, c0[c + 1])):
            print(f"  j={j-lo}: {T[j,0]} / {T[j,1]} / {T[j,2]} / {T[j,3]} ;",
                  " ".join(f"w{w}:{rs[j,w]},{dd[j,w]},{dn[j,w]}" for w in range(nw)))
    # handoff analysis: chunk (c, level L) vs producer chunk (c-1, level L-1)
    ls = np.asarray(p.schedule.level_starts)
    ip = np.asarray(p.schedule.inv_perm)
    C = len(c0) - 1
    per = (p.n + C - 1) // C
    own = np.minimum(ip // per, C - 1)
    lev_of_r = np.repeat(np.arange(len(ls) - 1), np.diff(ls))
    key = np.unique(own.astype(np.int64) * 100000 + lev_of_r)
    kc, kl = key // 100000, key % 100000
    if len(key) == len(T):
        idx = {(int(a), int(b)): i for i, (a, b) in enumerate(zip(kc, kl))}
        lat, slack = [], []
        for i in range(len(T)):
            src = idx.get((int(kc[i]) - 1, int(kl[i]) - 1))
            if src is None or T[i, 2] < 0:
                continue
            lat.append(T[i, 2] - last[src])       # halo complete - producer chunk done
            slack.append(T[i, 1] - last[src])     # waiter saw blob - producer done (<0: waiter was waiting)
        lat, slack = np.array(lat), np.array(slack)
        print("halo staged - producer chunk done (ns):", q(lat))
        print("waiter sees blob - producer done (ns): ", q(slack))
        w_wait = lat[slack < 0]
        print("  when the waiter was already polling:  ", q(w_wait))
    else:
        print("chunk keys", len(key), "!= chunks", len(T), "(split chunks): handoff analysis skipped")
    starts = np.array([rs[c0[c]].min() for c in range(len(c0) - 1) if c0[c + 1] > c0[c]])
    print("CTA first-chunk start offsets (us): p50 step %.3f" % (np.median(np.diff(starts)) / 1e3))


if __name__ == "__main__":
    main()
