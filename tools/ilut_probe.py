import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1606_00541_b200 as H
s = int(sys.argv[1]) if len(sys.argv) > 1 else 128
a = H.gen_reservoir7(s, s, s)
t0 = time.time(); f = H.ilut(a, 10, 1e-3); print("ilut", time.time() - t0, flush=True)
for name, fac, up in (("L", f.l, False), ("U", f.u, True)):
    p = (H.prepare_upper if up else H.prepare_lower)(fac)
    t = H.DeviceTri.create(p)
    info = t.info()
    b = torch.ones(p.n, dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
    for _ in range(3): t.solve(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): t.solve(b, x)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(name, {k: info[k] for k in ("nlev", "layout", "ctas", "chunks", "group", "groups", "rows_per_lane", "width", "ring", "halo_ring", "nnz")}, f"{ms:.3f} ms, {ms*1e3/info['nlev']:.2f} us/level", flush=True)
