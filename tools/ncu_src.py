"""Per-instruction stall samples from `ncu --page source --csv --print-source sass`
(diagnostics): python tools/ncu_src.py file.csv [--min 0.3] [--all]"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--min", type=float, default=0.3, help="percent of samples to print an instruction")
    ap.add_argument("--all", action="store_true")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    body = rows[2:]
    st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
    print(f"total samples {tot:.0f}")
    for r in body:
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ex = r[ix["Instructions Executed"]]
        if not args.all and smp < args.min / 100 * tot:
            continue
        reasons = sorted(((float(r[ix[h]] or 0), h[6:]) for h in st), reverse=True)[:3]
        rs = " ".join(f"{n}:{100*v/tot:.1f}" for v, n in reasons if v > 0)
        print(f"{r[0][-5:]} {100*smp/tot:5.1f}% ex={ex:>8s} {r[1].strip()[:60]:60s} {rs}")


if __name__ == "__main__":
    main()
