"""Summarise an ncu --page source --csv --print-source sass export: top SASS
instructions by warp-stall samples with their dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
agg = {h: sum(float(d[h] or 0) for d in data) for h in stalls}
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]} {v/tot*100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
top = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
for d in top:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    reasons = sorted(((float(d[h] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{d['Address']:>6} {s/tot*100:5.1f}%  {d['Source'][:60]:60s}  " + " ".join(f"{n}:{v/tot*100:.1f}" for v, n in reasons if v))
