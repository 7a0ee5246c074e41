"""BASELINE configs 3 and 5 on one B200 (diagnostics / coverage; results go to
profiles/configs_r01.md).

  C3  heterogeneous reservoir 7-pt, ILU(1) and ILUT(tau=1e-3, p=10) inside
      GMRES(30), b = A*1 (single block, as SURVEY 8(b) for the reference);
      parity anchor: 64^3 iteration counts of the reference (ilu0 210, ilu1 73,
      ilut 424).
  C5  trisolve sweep: 7-pt grids 100^3 .. 256^3, natural / RCM / random
      orderings (level count vs rows per level), and fixed ELL widths 4-32.

python tools/config_sweep.py --c3 64 192 --c5
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def timed_lu(pl, pu, b, reps=5):
    import torch
    tl, tu = H.DeviceTri.create(pl), H.DeviceTri.create(pu)
    bd = torch.tensor(b, device="cuda")
    y, x = torch.empty_like(bd), torch.empty_like(bd)
    for _ in range(2):
        tl.solve(bd, y)
        tu.solve(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        e0.record()
        tl.solve(bd, y)
        tu.solve(y, x)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    alg = tl.info()["alg_bytes"] + tu.info()["alg_bytes"]
    return float(np.median(ms)), alg, tl.info()


def c3(size, out):
    a = H.gen_reservoir7(size, size, size)
    b = H.spmv_csr(a, np.ones(a.n_rows), workers=os.cpu_count())
    for name, kind, kw in (("ilu0", "bilu0", {}), ("ilu1", "biluk", {"fill_level": 1}),
                           ("ilut(10,1e-3)", "bilut", {"ilut_p": 10, "ilut_tol": 1e-3})):
        t0 = time.time()
        m = H.build_preconditioner(a, kind, 1, 0, **kw)
        setup = time.time() - t0
        res = H.gmres(a, b, m, H.SolverConfig(restart=30))
        li, ui = m.device_info() if hasattr(m, "device_info") else (None, None)
        rec = dict(config="C3", size=size, precond=name, iterations=res.report.iterations,
                   converged=res.report.converged, rel=res.report.final_relative_residual,
                   solve_s=round(res.report.solve_seconds, 4), setup_s=round(setup, 1),
                   max_err=float(np.max(np.abs(res.x - 1.0))),
                   nlev=(m.prepared_l.schedule.nlev, m.prepared_u.schedule.nlev),
                   ell_width=(m.prepared_l.hec.ell.width, m.prepared_u.hec.ell.width))
        print(json.dumps(rec), flush=True)
        out.append(rec)


def c5(out):
    for s in (100, 128, 160, 202, 256):
        a = H.gen_poisson7(s, s, s)
        b = H.spmv_csr(a, np.ones(a.n_rows), workers=os.cpu_count())
        orders = [("natural", None)]
        if s <= 128:
            orders += [("rcm", H.rcm_ordering(a)), ("random", H.random_ordering(a.n_rows, 1606))]
        for oname, perm in orders:
            ap = a if perm is None else H.permute_symmetric(a, perm)
            bp = b if perm is None else H.spmv_csr(ap, np.ones(a.n_rows), workers=os.cpu_count())
            f = H.ilu0(ap)
            pl, pu = H.prepare_lower(f.l), H.prepare_upper(f.u)
            ms, alg, info = timed_lu(pl, pu, bp)
            rec = dict(config="C5", grid=f"7pt {s}^3", ordering=oname, n=a.n_rows, nlev=pl.schedule.nlev,
                       rows_per_level=round(a.n_rows / pl.schedule.nlev), ms_LU=round(ms, 4),
                       GBs=round(alg / ms / 1e6, 1), layout_ctas=info["ctas"])
            print(json.dumps(rec), flush=True)
            out.append(rec)
    # ELL width sweep (fixed widths; 27-pt: 13 eligible per row, w<13 spills to the CSR tail)
    for st, s in ((27, 96), (7, 128)):
        a = H.gen_poisson27(s, s, s) if st == 27 else H.gen_poisson7(s, s, s)
        b = H.spmv_csr(a, np.ones(a.n_rows), workers=os.cpu_count())
        f = H.ilu0(a)
        for w in (4, 8, 16, 32):
            pl = H.prepare_lower(f.l, H.WidthPolicy.fixed(w))
            pu = H.prepare_upper(f.u, H.WidthPolicy.fixed(w))
            ms, alg, info = timed_lu(pl, pu, b)
            rec = dict(config="C5-width", grid=f"{st}pt {s}^3", ell_width=w, ms_LU=round(ms, 4),
                       GBs=round(alg / ms / 1e6, 1))
            print(json.dumps(rec), flush=True)
            out.append(rec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", type=int, nargs="*", default=[])
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--out", default="gpurun_out/configs.json")
    args = ap.parse_args()
    out = []
    for s in args.c3:
        c3(s, out)
    if args.c5:
        c5(out)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
