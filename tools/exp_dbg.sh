cat > /tmp/b.py <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1606_00541_b200 as H
for st, s in ((27, 128), (7, 256)):
    a = H.gen_poisson27(s, s, s) if st == 27 else H.gen_poisson7(s, s, s)
    f = H.ilu0(a)
    tl, tu = H.DeviceTri.create(H.prepare_lower(f.l)), H.DeviceTri.create(H.prepare_upper(f.u))
    b = torch.tensor(H.spmv_csr(a, np.ones(a.n_rows)), device="cuda")
    y, x = torch.empty_like(b), torch.empty_like(b)
    for _ in range(3): tl.solve(b, y); tu.solve(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(10):
        e0.record(); tl.solve(b, y); tu.solve(y, x); e1.record(); e1.synchronize(); ms.append(e0.elapsed_time(e1))
    print(f"{os.environ.get('TAG','')} {st}-pt {s}^3 L+U (b=A*1) {np.median(ms):.4f} ms", flush=True)
PY
for d in 0 2; do TAG="dbg=$d" HEC_WAVE_DBG=$d python /tmp/b.py; done
