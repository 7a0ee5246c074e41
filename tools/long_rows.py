"""Long CSR rows (diagnostics): lower-triangular factors whose rows mostly have a
few dependencies but some have thousands (an arrow-like tail, the loop at
proj/src/triangular.cpp:123-125), solved by the level launches and by the
wavefront kernel; prints the solve time per strategy (bitwise parity of the
warp rows: tests/test_gpu_trisolve.py::test_warp_rows_bitwise).

    python tools/long_rows.py --n 400000 --levels 4 --long-every 256 --long-len 4096
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def long_row_factor(n, levels, long_every, long_len, seed=0):
    """Rows split into `levels` bands; a row of band k>0 depends on 3 random rows
    of band k-1, every `long_every`-th row on `long_len` rows of earlier bands."""
    rng = np.random.default_rng(seed)
    band = n // levels
    rp, ci, vv = [0], [], []
    for i in range(n):
        k = i // band
        if k == 0 or k >= levels:
            cols = np.zeros(0, np.int64)
        else:
            lo = (k - 1) * band
            m = long_len if i % long_every == 0 else 3
            m = min(m, k * band)
            cols = np.unique(rng.integers(0, k * band, m) if m > 3 else rng.integers(lo, lo + band, m))
        vals = rng.uniform(-1, 1, cols.size) / max(cols.size, 1)
        ci.append(cols)
        ci.append(np.array([i]))
        vv.append(vals)
        vv.append(np.array([1.5 + rng.uniform()]))
        rp.append(rp[-1] + cols.size + 1)
    return np.array(rp, np.int64), np.concatenate(ci), np.concatenate(vv)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=400000)
    ap.add_argument("--levels", type=int, default=4)
    ap.add_argument("--long-every", type=int, default=256)
    ap.add_argument("--long-len", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    t0 = time.time()
    rp, ci, vv = long_row_factor(args.n, args.levels, args.long_every, args.long_len)
    m = H.CsrMatrix.from_arrays(args.n, args.n, rp, ci, vv)
    p = H.prepare_lower(m)
    print(f"n {args.n} nnz {len(vv)} levels {p.schedule.nlev} setup {time.time() - t0:.1f} s", flush=True)
    b = np.random.default_rng(1).uniform(-1, 1, args.n)
    for strategy in (0, 1, 2):  # auto, level launches, wavefront
        try:
            t = H.DeviceTri.create(p, strategy=strategy)
        except Exception as e:  # noqa: BLE001
            print(f"strategy {strategy}: {e}")
            continue
        info = t.info()
        bd = torch.tensor(b, device="cuda")
        x = torch.empty_like(bd)
        for _ in range(3):
            t.solve(bd, x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(args.reps):
            e0.record()
            t.solve(bd, x)
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        print(f"asked {strategy}: strategy {info['strategy']} layout {info.get('layout')}: {np.median(ms):.4f} ms", flush=True)
        del t


if __name__ == "__main__":
    main()
