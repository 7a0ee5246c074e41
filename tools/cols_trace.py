"""Column-kernel trace (diagnostics): per CTA, when its first level finished, its
per-level period, and how often its edge lanes had to re-poll a mailbox.

    python tools/cols_trace.py 7:256 [--which L|U]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("grid")
    ap.add_argument("--which", default="L")
    args = ap.parse_args()
    import torch
    st, s = (int(v) for v in args.grid.split(":"))
    a = H.gen_poisson7(s, s, s)
    f = H.ilu0(a)
    p = H.prepare_lower(f.l) if args.which == "L" else H.prepare_upper(f.u)
    t = H.DeviceTri.create(p, strategy=2)
    info = t.info()
    print(info)
    b = torch.ones(p.n, dtype=torch.float64, device="cuda")
    x = torch.empty_like(b)
    for _ in range(3):
        t.solve(b, x)
    tr, c0 = t.solve_traced(b, x)
    tr = tr.reshape(-1)[: 8 * info["chunks"]].reshape(-1, 8).astype(np.int64)
    end, start, loaded = tr[:, 0], tr[:, 3], tr[:, 2]
    pl, pd = tr[:, 1] & 0xffffffff, tr[:, 1] >> 32
    T0 = start[start > 0].min()
    ncta = len(c0) - 1
    first, last, per, polls, busy = [], [], [], [], []
    for c in range(ncta):
        e = end[c0[c]:c0[c + 1]] - T0
        b0 = start[c0[c]:c0[c + 1]] - T0
        first.append(e[0])
        last.append(e[-1])
        d = np.diff(e)
        per.append(np.median(d) if len(d) else 0)
        polls.append(int(pl[c0[c]:c0[c + 1]].sum() + pd[c0[c]:c0[c + 1]].sum()))
        busy.append(np.median(e - b0))
    first, last, per = np.array(first), np.array(last), np.array(per)
    print(f"solve {last.max() / 1e3:.1f} us; CTA first level done: min {first.min() / 1e3:.2f} max "
          f"{first.max() / 1e3:.2f} us; last: min {last.min() / 1e3:.1f} max {last.max() / 1e3:.1f} us")
    print(f"per-level period (median per CTA) p10 {np.percentile(per, 10):.0f} p50 {np.median(per):.0f} "
          f"p90 {np.percentile(per, 90):.0f} ns; level start->end p50 {np.median(busy):.0f} ns")
    ld = loaded - start
    st = tr[:, 4:8]
    ok = st[:, 3] > 0
    ok[c0[1]:] = False  # CTA 0 only: no mailbox waits
    if ok.any(): print("warp 0 SM-clock stamps from level start (cycles, p50): " + ", ".join(
        f"{n} {np.median(st[ok, i]):.0f}" for i, n in enumerate(("data ready", "data loaded", "x", "published"))) +
        f", level end {np.median(tr[ok, 2]):.0f}")
    print(f"mailbox re-polls per CTA: p50 {np.median(polls):.0f} max {max(polls)}; total {sum(polls)}")
    order = np.argsort(first)
    for c in order[:: max(1, ncta // 12)]:
        e = end[c0[c]:c0[c + 1]] - T0
        d = np.diff(e)
        print(f"  cta {c:3d}: levels {c0[c + 1] - c0[c]:4d} first {e[0] / 1e3:7.2f} us last {e[-1] / 1e3:7.1f} us "
              f"period p50 {np.median(d):.0f} p90 {np.percentile(d, 90):.0f} ns polls "
              f"{int(pl[c0[c]:c0[c + 1]].sum())}/{int(pd[c0[c]:c0[c + 1]].sum())}")


if __name__ == "__main__":
    main()
