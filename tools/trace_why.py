"""Why is each chunk late? (diagnostics, traced k_wave)

For every chunk j of every CTA: start_j = max(ready_j, done_{j-1}) where ready_j is
the waiter's publish time (foreign values staged) and done_{j-1} the previous
chunk's completion in the same CTA (the named-barrier hand-off). Reports, over
all chunks: how often the chunk waited for its halo (ready > prev done) vs for
its own predecessor, the compute time done_j - start_j, the blob latency
(landed - issued), and the active-CTA profile over time.

    python tools/trace_why.py --stencil 7 --size 256 [--which L]
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
    ap.add_argument("--which", default="L")
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s) if args.stencil == "7" else H.gen_poisson27(s, s, s)
    f = H.ilu0(a)
    p = H.prepare_lower(f.l) if args.which == "L" else H.prepare_upper(f.u)
    t = H.DeviceTri.create(p, strategy=2)
    b = torch.ones(p.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(3):
        t.solve(b, x)
    tr, c0 = t.solve_traced(b, x)
    tr = tr.astype(np.int64)
    info = t.info()
    nw = info["group"] * info["groups"]  # solver warps
    T0 = tr[:, 0][tr[:, 0] > 0].min()
    T = np.where(tr > 0, tr - T0, -1)
    issued, landed, ready = T[:, 0], T[:, 1], T[:, 3]
    done = T[:, 10:10 + 3 * nw:3].max(axis=1)
    ncta = len(c0) - 1
    halo_bound = comp = lat = 0
    comp_t, halo_gap, own_gap, land_lat = [], [], [], []
    first, last = np.zeros(ncta), np.zeros(ncta)
    for c in range(ncta):
        lo, hi = c0[c], c0[c + 1]
        first[c], last[c] = done[lo], done[hi - 1]
        prev = -1
        for j in range(lo, hi):
            start = max(ready[j], prev) if prev >= 0 else ready[j]
            if prev >= 0:
                if ready[j] > prev:
                    halo_bound += 1
                    halo_gap.append(ready[j] - prev)
                else:
                    own_gap.append(prev - ready[j])
            comp_t.append(done[j] - start)
            land_lat.append(landed[j] - issued[j])
            prev = done[j]
    total = done.max()
    print(f"{args.stencil}-pt {s}^3 {args.which}: {ncta} CTAs, {len(done)} chunks, solve {total/1e3:.1f} us "
          f"(layout {info.get('layout')}, shape {info.get('group')}x{info.get('groups')}x{info.get('rows_per_lane')})")
    n = len(done) - ncta
    print(f"chunks that waited for their halo (ready after prev done): {halo_bound}/{n} = {100*halo_bound/max(n,1):.1f}%"
          f", median halo gap {np.median(halo_gap) if halo_gap else 0:.0f} ns")
    print(f"compute (done - start): p50 {np.percentile(comp_t,50):.0f} p90 {np.percentile(comp_t,90):.0f} ns; "
          f"blob latency (landed - issued) p50 {np.percentile(land_lat,50):.0f} ns")
    print(f"CTA first-chunk done: min {first.min()/1e3:.1f} max {first.max()/1e3:.1f} us; last: min {last.min()/1e3:.1f} "
          f"max {last.max()/1e3:.1f} us")
    per = [(done[c0[c + 1] - 1] - done[c0[c]]) / max(c0[c + 1] - c0[c] - 1, 1) for c in range(ncta)]
    print(f"per-CTA chunk period: p10 {np.percentile(per,10):.0f} p50 {np.percentile(per,50):.0f} "
          f"p90 {np.percentile(per,90):.0f} ns")
    # chunk period (done_j - done_{j-1}) of chunks whose halo was staged before the
    # previous chunk finished, by rows in the chunk: flat = latency chain, rising = throughput
    rows = tr[:, 7]
    per_rows = {}
    for c in range(ncta):
        for j in range(c0[c] + 1, c0[c + 1]):
            if ready[j] <= done[j - 1]:
                per_rows.setdefault(int(rows[j]) // 64, []).append(done[j] - done[j - 1])
    print("own-bound chunk period by rows (64-row bins): " + ", ".join(
        f"{64 * k}-{64 * k + 63}: p50 {np.median(v):.0f} ns (n={len(v)})" for k, v in sorted(per_rows.items())))
    # parts of the own-bound period: prefetch done (words 56..), barrier passed (9+3w), done
    gmax = min(info.get("group") or 1, 8)
    pre = np.where(T[:, 56:56 + gmax] >= 0, T[:, 56:56 + gmax], -1).max(axis=1)
    bar = T[:, 9:9 + 3 * nw:3].max(axis=1)
    parts = {"prefetch_done - prev_done": [], "barrier - prev_done": [], "done - barrier": [],
             "ready - prev_done": [], "landed - prev_done": []}
    for c in range(ncta):
        for j in range(c0[c] + 1, c0[c + 1]):
            if ready[j] <= done[j - 1]:
                parts["prefetch_done - prev_done"].append(pre[j] - done[j - 1])
                parts["barrier - prev_done"].append(bar[j] - done[j - 1])
                parts["done - barrier"].append(done[j] - bar[j])
                parts["ready - prev_done"].append(ready[j] - done[j - 1])
                parts["landed - prev_done"].append(landed[j] - done[j - 1])
    for k, v in parts.items():
        print(f"  own-bound {k}: p10 {np.percentile(v, 10):.0f} p50 {np.median(v):.0f} p90 {np.percentile(v, 90):.0f} ns")
    st = tr[:, 48:54].astype(np.int64)
    # warp 0 (group 0) stamps its chunks only: local chunk index divisible by the group count
    K = max(info.get("groups") or 1, 1)
    local = np.concatenate([np.arange(c0[c + 1] - c0[c]) for c in range(ncta)])
    sel = (local % K == 0) & (st[:, 1] > 0)
    if sel.any():
        print("  warp-0 SM-clock stamps after its barrier (cycles, p50): " + ", ".join(
            f"{n} {np.median(st[sel, k]):.0f}" for k, n in ((1, "gathers"), (2, "fp"), (3, "stores"),
                                                            (4, "bar.arrive"), (5, "x stores"))))
    bins = np.linspace(0, total, 11)
    act = [int(np.sum((first <= b1) & (last >= b0))) for b0, b1 in zip(bins[:-1], bins[1:])]
    print("active CTAs per tenth of the solve:", act)


if __name__ == "__main__":
    main()
