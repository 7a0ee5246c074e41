"""Per-CTA start lag and chunk period from the traced kernel (diagnostics).
python tools/cta_lag.py --stencil 27 --size 128"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stencil", default="27")
    ap.add_argument("--size", type=int, default=128)
    args = ap.parse_args()
    import torch
    s = args.size
    a = H.gen_poisson7(s, s, s) if args.stencil == "7" else H.gen_poisson27(s, s, s)
    p = H.prepare_lower(H.ilu0(a).l)
    t = H.DeviceTri.create(p, strategy=2)
    b = torch.tensor(H.spmv_csr(a, np.ones(a.n_rows)), device="cuda")
    x = torch.empty_like(b)
    for _ in range(3):
        t.solve(b, x)
    tr, c0 = t.solve_traced(b, x)
    tr = tr.astype(np.int64)
    info = t.info()
    nw = info["group"] * info["groups"]  # solver warps
    T = np.where(tr > 0, tr - tr[:, 0].min(), -1)
    done = T[:, 10:10 + 3 * nw:3].max(axis=1)
    C = len(c0) - 1
    first = np.array([done[c0[c]] for c in range(C)])
    last = np.array([done[c0[c + 1] - 1] for c in range(C)])
    per = np.array([np.median(np.diff(done[c0[c]:c0[c + 1]])) for c in range(C)])
    print(f"{C} CTAs, span {last.max()/1e3:.1f} us; first-chunk done: CTA0 {first[0]/1e3:.2f} us, "
          f"median step {np.median(np.diff(first))/1e3:.3f} us; chunk period p50 over CTAs {np.median(per):.0f} ns "
          f"(CTA0 {per[0]:.0f}); busy span per CTA p50 {np.median(last-first)/1e3:.1f} us")
    for c in (0, 1, 2, 10, C // 2, C - 1):
        n = c0[c + 1] - c0[c]
        print(f"  CTA {c}: {n} chunks, first done {first[c]/1e3:.2f} us, last {last[c]/1e3:.2f} us, period {per[c]:.0f} ns")


if __name__ == "__main__":
    main()
