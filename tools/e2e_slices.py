"""End-to-end ILU apply through the C-ABI host entry (hec_precond_apply_host,
pinned host buffers) against the number of host-copy slices (HEC_HOST_SLICES),
interleaved rounds, median per call; plus the bare PCIe copy times.

    python tools/e2e_slices.py --grid 256 --slices 1,2,4,8 --rounds 5
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--slices", default="1,2,4,8")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--calls", type=int, default=10)
    args = ap.parse_args()
    import torch
    s = args.grid
    a = H.gen_poisson7(s, s, s)
    f = H.ilu0(a)
    n = a.n_rows
    dp = H.DevicePrecond.create(n, H.prepare_lower(f.l), H.prepare_upper(f.u))
    bh = torch.empty(n, dtype=torch.float64).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    bh.numpy()[:] = np.random.default_rng(0).uniform(-1, 1, n)
    pb, px = bh.numpy().ctypes.data_as(H.api.L.P_dbl), xh.numpy().ctypes.data_as(H.api.L.P_dbl)

    def call():
        H.api.check(H.api.lib.hec_precond_apply_host(dp._h, pb, px))

    ref = None
    times = {k: [] for k in args.slices.split(",")}
    for _ in range(args.rounds):
        for k in times:
            os.environ["HEC_HOST_SLICES"] = k
            call()
            if ref is None:
                ref = xh.numpy().copy()
            assert (xh.numpy().view(np.uint64) == ref.view(np.uint64)).all(), k
            for _ in range(args.calls):
                t0 = time.perf_counter()
                call()
                times[k].append((time.perf_counter() - t0) * 1e3)
    for k, v in times.items():
        print(f"{s}^3 slices {k}: median {np.median(v):.3f} ms, min {np.min(v):.3f} ms ({len(v)} calls)", flush=True)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for name, fn in (("H2D", lambda: d.copy_(bh, non_blocking=True)), ("D2H", lambda: xh.copy_(d, non_blocking=True))):
        ms = []
        for _ in range(10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ms.append((time.perf_counter() - t0) * 1e3)
        print(f"bare {name} {8 * n / 1e6:.0f} MB: median {np.median(ms):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
