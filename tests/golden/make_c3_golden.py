"""BASELINE config C3 goldens from the REFERENCE itself (oracle/_ref/libhecref.so):
GMRES(30) iteration counts on the heterogeneous reservoir-style 7-point matrix
(gen_reservoir7, sigma 3, kz_ratio 0.1, seed 1606; the
matrix comes from the C oracle's restatement oracle/hec_oracle.c:orc_reservoir7,
not from the product), b = A*1 (bench.cpp:110-111), rel_tol 1e-6, one block
holding ilu0 / ilu_k(1) / ilut(10, 1e-3) factors (the SURVEY.md 8(b)
hand-assembled single-block preconditioner; PrecondKind has no ILU(k)).

    make -C oracle && python tests/golden/make_c3_golden.py [--sizes 64 192] [--workers 4]

Writes tests/golden/c3_gmres.json (one entry per size and factor kind,
appended as each run finishes, so a long 192^3 sweep can be resumed).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import load_oracle, load_reference  # noqa: E402

OUT = os.path.join(HERE, "c3_gmres.json")
KINDS = (("ilu0", "ilu0", 0, 0.0), ("ilu1", "iluk", 1, 0.0), ("ilut", "ilut", 10, 1e-3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[64, 192])
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--kinds", nargs="+", default=[k[0] for k in KINDS])
    args = ap.parse_args()
    ref, orc = load_reference(), load_oracle()
    if ref is None:
        raise SystemExit("oracle/_ref/libhecref.so not built")
    done = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for size in args.sizes:
        a = orc.reservoir7(size, size, size)
        b = ref.spmv(a, np.ones(a.n), args.workers)
        for name, kind, k, tol in KINDS:
            key = f"{size}_{name}"
            if name not in args.kinds or key in done:
                continue
            t0 = time.time()
            l, u = ref.ilu(a, kind, k, tol)
            m = ref.precond_single(l, u)
            t1 = time.time()
            x, rep = ref.gmres(a, b, m, restart=30, max_iters=10000, rel_tol=1e-6, workers=args.workers)
            done[key] = {"size": size, "factor": name, "iterations": rep["iterations"],
                         "converged": rep["converged"], "final_relative_residual": float(rep["final_relative_residual"]),
                         "max_abs_error_vs_ones": float(np.max(np.abs(x - 1.0))),
                         "nnz_l": int(l.rp[-1]), "nnz_u": int(u.rp[-1]), "setup_seconds": round(t1 - t0, 1),
                         "gmres_seconds": round(float(rep["solve_seconds"]), 1), "workers": args.workers,
                         "restart": 30, "rel_tol": 1e-6}
            print(key, done[key], flush=True)
            with open(OUT, "w") as f:
                json.dump(done, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
