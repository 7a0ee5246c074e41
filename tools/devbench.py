"""Developer timing of the trisolve strategies (not the bench contract).

python tools/devbench.py --grid 7:256 --grid 27:128 --ctas 148 --reps 10
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
    ap.add_argument("--grid", action="append", default=[])
    ap.add_argument("--ctas", type=int, nargs="*", default=[0])
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--strategies", type=int, nargs="*", default=[1, 2])
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    import torch
    torch.cuda.init()
    for g in args.grid or ["7:128"]:
        st, size = g.split(":")
        size = int(size)
        t0 = time.time()
        a = H.gen_poisson7(size, size, size) if st == "7" else H.gen_poisson27(size, size, size)
        f = H.ilu0(a)
        t1 = time.time()
        pl = H.prepare_lower(f.l)
        pu = H.prepare_upper(f.u)
        t2 = time.time()
        print(f"# {st}-pt {size}^3 n={a.n_rows} nnzL={f.l.nnz()} nlev={pl.schedule.nlev}/{pu.schedule.nlev} "
              f"w={pl.hec.ell.width} gen+ilu0 {t1-t0:.1f}s prepare {t2-t1:.1f}s", flush=True)
        n = a.n_rows
        b = torch.ones(n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(b)
        x = torch.empty_like(b)
        ref_x = None
        for strat in args.strategies:
            for ctas in (args.ctas if strat == 2 else [0]):
                tb = time.time()
                tl = H.DeviceTri.create(pl, strategy=strat, ctas=ctas, threads=args.threads)
                tu = H.DeviceTri.create(pu, strategy=strat, ctas=ctas, threads=args.threads)
                tc = time.time() - tb
                il, iu = tl.info(), tu.info()
                stream = torch.cuda.current_stream()
                for _ in range(3):
                    tl.solve(b, y, stream)
                    tu.solve(y, x, stream)
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                tl_ms, tu_ms = [], []
                for _ in range(args.reps):
                    ev[0].record(stream)
                    tl.solve(b, y, stream)
                    ev[1].record(stream)
                    tu.solve(y, x, stream)
                    ev[2].record(stream)
                    ev[2].synchronize()
                    tl_ms.append(ev[0].elapsed_time(ev[1]))
                    tu_ms.append(ev[1].elapsed_time(ev[2]))
                ms = np.median(np.array(tl_ms) + np.array(tu_ms))
                alg = il["alg_bytes"] + iu["alg_bytes"]
                xs = x.cpu().numpy()
                if ref_x is None:
                    ref_x = xs
                same = bool((xs.view(np.uint64) == ref_x.view(np.uint64)).all())
                print(f"strategy={strat} ctas={il['ctas']} thr={il['threads']} chunks={il['chunks']} "
                      f"L {np.median(tl_ms):.3f} ms U {np.median(tu_ms):.3f} ms L+U {ms:.3f} ms "
                      f"{alg/ms/1e6:.1f} GB/s ({alg/ms/1e6/6545.6*100:.1f}% of 6545.6) build {tc:.1f}s "
                      f"same_as_first={same}", flush=True)
                del tl, tu


if __name__ == "__main__":
    main()
