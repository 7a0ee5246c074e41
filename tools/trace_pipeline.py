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
    t0 = tr[:, 0].min()
    T = tr - t0
    T[:, 7] = tr[:, 7]
    end = T[:, 5].max()
    print(f"chunks {len(T)}  span {end/1e3:.1f} us (first blob issue -> last publish)")
    names = ["issue", "gather", "wstart", "cleared", "sstart", "sdone", "publish"]
    print("blob issue -> gather issue (ns):   ", q(T[:, 1] - T[:, 0]))
    print("gather -> waiter start:            ", q(T[:, 2] - T[:, 1]))
    print("waiter poll (start -> cleared):    ", q(T[:, 3] - T[:, 2]))
    print("cleared -> solvers start:          ", q(T[:, 4] - T[:, 3]))
    print("solvers compute (start -> done):   ", q(T[:, 5] - T[:, 4]))
    print("solver SM cycles:                  ", q(T[:, 7]))
    print("  cycles to header decoded:        ", q(tr[:, 8]))
    print("  cycles to acc (row 0):           ", q(tr[:, 9]))
    print("  cycles to x (after div):         ", q(tr[:, 10]))
    print("  cycles to rows done (thread 0):  ", q(tr[:, 11]))
    # solver idle gap between consecutive chunks of one CTA
    gaps, busy, first_start, last_done = [], [], [], []
    for c in range(len(c0) - 1):
        lo, hi = c0[c], c0[c + 1]
        if hi <= lo:
            continue
        st, dn = T[lo:hi, 4], T[lo:hi, 5]
        gaps.extend((st[1:] - dn[:-1]).tolist())
        busy.append((dn - st).sum())
        first_start.append(st[0])
        last_done.append(dn[-1])
    print("solver gap between chunks (ns):    ", q(gaps))
    busy = np.array(busy)
    span = np.array(last_done) - np.array(first_start)
    print(f"per-CTA busy fraction: mean {np.mean(busy / np.maximum(span, 1)):.3f}; "
          f"first start p50 {np.median(first_start)/1e3:.1f} us, last done p50 {np.median(last_done)/1e3:.1f} us")
    # where does the gap go: waiting for the waiter (cross-CTA) or for data (producer)?
    wait_cross = T[:, 3] - np.maximum(T[:, 2], 0)
    print("gap attributable to cross-CTA wait (cleared - wstart) when solvers idle:")
    idle_cross, idle_data = [], []
    for c in range(len(c0) - 1):
        lo, hi = c0[c], c0[c + 1]
        for j in range(lo + 1, hi):
            gap_start = T[j - 1, 5]
            if T[j, 4] - gap_start < 200:
                continue
            # data ready at T[j,2] (waiter saw full+ready), cross cleared at T[j,3]
            idle_data.append(max(0, T[j, 2] - gap_start))
            idle_cross.append(max(0, T[j, 3] - max(T[j, 2], gap_start)))
    print("   data (producer) part:   ", q(idle_data))
    print("   cross-CTA wait part:    ", q(idle_cross))
    # per-CTA detail (ticket order == owner order)
    print("cta  chunks  first_start  last_done  us/chunk  busy%  mean_gap  wstart->cleared  cleared->start")
    for c in sorted(set([0, 1, 2, 3, 5, 10, 30, 70, 110, len(c0) - 2])):
        lo, hi = c0[c], c0[c + 1]
        if hi <= lo:
            continue
        st, dn = T[lo:hi, 4], T[lo:hi, 5]
        span = dn[-1] - st[0]
        busy = (dn - st).sum()
        print(f"{c:4d} {hi-lo:6d} {st[0]/1e3:11.1f} {dn[-1]/1e3:10.1f} {span/(hi-lo)/1e3:9.2f} {100*busy/max(span,1):6.1f} "
              f"{np.mean(st[1:]-dn[:-1]) if hi-lo>1 else 0:9.0f} {np.median(T[lo:hi,3]-T[lo:hi,2]):15.0f} "
              f"{np.median(T[lo:hi,4]-T[lo:hi,3]):14.0f}")


if __name__ == "__main__":
    main()
