# mailbox poll back-off sweep (HEC_WAVE_SPIN_NS), ILU apply time with b = A*1
cat > /tmp/spin.py <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1606_00541_b200 as H
for st, s in ((27, 128), (7, 256)):
    a = H.gen_poisson27(s, s, s) if st == 27 else H.gen_poisson7(s, s, s)
    f = H.ilu0(a)
    dp = H.DevicePrecond.create(a.n_rows, H.prepare_lower(f.l), H.prepare_upper(f.u))
    b = torch.tensor(H.spmv_csr(a, np.ones(a.n_rows)), device="cuda")
    x = torch.empty_like(b)
    for _ in range(3): dp.apply(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(10):
        e0.record(); dp.apply(b, x); e1.record(); e1.synchronize(); ms.append(e0.elapsed_time(e1))
    print(f"spin={os.environ.get('HEC_WAVE_SPIN_NS','0')} {st}-pt {s}^3 ILU apply {np.median(ms):.4f} ms", flush=True)
PY
for v in 0 32 128 512; do HEC_WAVE_SPIN_NS=$v python /tmp/spin.py; done
