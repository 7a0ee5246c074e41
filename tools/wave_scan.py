"""Wave-kernel scan (diagnostics): solve time of one factor against the CTA count
and solver shape, to tell a latency-bound chunk chain (time flat in the rows per
chunk) from a throughput-bound one (time growing with the rows per chunk).

    python tools/wave_scan.py 7:256 --which L --ctas 143,96,64,32 --shapes 8x2x2,4x2x4
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_00541_b200 as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("grids", nargs="+")
    ap.add_argument("--which", default="L")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--shapes", default="")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    for g in args.grids:
        st, s = (int(v) for v in g.split(":"))
        a = H.gen_poisson27(s, s, s) if st == 27 else H.gen_poisson7(s, s, s)
        f = H.ilu0(a)
        p = H.prepare_lower(f.l) if args.which == "L" else H.prepare_upper(f.u)
        nnz = p.hec.ell.width * p.n
        for shape in (args.shapes.split(",") if args.shapes else [""]):
            if shape:
                G, K, R = shape.split("x")
                os.environ.update(HEC_WAVE_G=G, HEC_WAVE_K=K, HEC_WAVE_RPL=R)
            for c in (int(v) for v in args.ctas.split(",")):
                try:
                    t = H.DeviceTri.create(p, strategy=2, ctas=c)
                except Exception as e:  # noqa: BLE001
                    print(f"{st}-pt {s}^3 {args.which} shape {shape or 'auto'} ctas {c}: {e}")
                    continue
                info = t.info()
                bp = torch.ones(info["wave_len"] + 2, dtype=torch.float64, device="cuda")
                xw = torch.empty(info["wave_len"], dtype=torch.float64, device="cuda")
                for _ in range(3):
                    t.solve_wave(bp, xw)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ms = []
                for _ in range(args.reps):
                    e0.record()
                    t.solve_wave(bp, xw)
                    e1.record()
                    e1.synchronize()
                    ms.append(e0.elapsed_time(e1))
                m = float(np.median(ms))
                rows_per_chunk = p.n / max(info["chunks"], 1)
                per_chunk_ns = m * 1e6 / max(info["chunks"] / max(info["ctas"], 1), 1)
                print(f"{st}-pt {s}^3 {args.which} shape {shape or 'auto'} ({info.get('group')}x{info.get('groups')}x"
                      f"{info.get('rows_per_lane')}) ctas {info['ctas']} layout {info.get('layout')}: {m:.4f} ms, "
                      f"chunks {info['chunks']} ({rows_per_chunk:.0f} rows avg), levels {p.schedule.nlev}, "
                      f"{m * 1e6 / p.schedule.nlev:.0f} ns/level, {per_chunk_ns:.0f} ns per CTA chunk, "
                      f"{12 * (nnz + p.n) + 20 * p.n:.3g} B", flush=True)
                del t
            for k in ("HEC_WAVE_G", "HEC_WAVE_K", "HEC_WAVE_RPL"):
                os.environ.pop(k, None)


if __name__ == "__main__":
    main()
