"""Stall / parity stress of the wave kernel across layouts (diagnostics):
many solves per configuration with a per-solve watchdog and a bitwise check
against the first result.  python tools/stress.py --n 300"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=300)
    args = ap.parse_args()
    import torch
    import paper_1606_00541_b200 as H
    cases = []
    for s in (24, 61, 128):
        cases.append((f"7pt {s}^3 ilu0", H.gen_poisson7(s, s, s), None, "ilu0"))
    cases.append(("27pt 64^3 ilu0", H.gen_poisson27(64, 64, 64), None, "ilu0"))
    cases.append(("7pt 64^3 rcm ilu0", H.gen_poisson7(64, 64, 64), "rcm", "ilu0"))
    cases.append(("7pt 48^3 random ilu0", H.gen_poisson7(48, 48, 48), "random", "ilu0"))
    cases.append(("27pt 40^3 ilu1", H.gen_poisson27(40, 40, 40), None, "ilu1"))
    cases.append(("reservoir 48^3 ilut", H.gen_reservoir7(48, 48, 48), None, "ilut"))
    rng = np.random.default_rng(5)
    bad = 0
    for name, a, order, kind in cases:
        if order == "rcm":
            a = H.permute_symmetric(a, H.rcm_ordering(a))
        elif order == "random":
            a = H.permute_symmetric(a, H.random_ordering(a.n_rows, 7))
        f = H.ilu0(a) if kind == "ilu0" else (H.ilu_k(a, 1) if kind == "ilu1" else H.ilut(a, 10, 1e-3))
        dp = H.DevicePrecond.create(a.n_rows, H.prepare_lower(f.l), H.prepare_upper(f.u))
        b = torch.tensor(rng.uniform(-1, 1, a.n_rows), device="cuda")
        x = torch.empty_like(b)
        dp.apply(b, x)
        torch.cuda.synchronize()
        ref = x.clone()
        t0 = time.time()
        for k in range(args.n):
            x.fill_(float("nan"))
            t1 = time.time()
            dp.apply(b, x)
            ev = torch.cuda.Event()
            ev.record()
            while not ev.query():
                if time.time() - t1 > 10:
                    print(f"STALL {name} at solve {k}", flush=True)
                    os._exit(3)
            if k % 50 == 0 and not torch.equal(x.view(torch.int64), ref.view(torch.int64)):
                print(f"MISMATCH {name} at solve {k}", flush=True)
                bad += 1
        print(f"{name}: {args.n} applies ok in {time.time()-t0:.2f}s", flush=True)
    print("stress done, mismatches", bad, flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
