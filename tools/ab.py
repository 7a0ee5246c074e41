"""A/B timing of the ILU apply between two builds of the package (diagnostics):
python tools/ab.py <package parent dir> 27:128 7:256"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.abspath(sys.argv[1]))
import paper_1606_00541_b200 as H  # noqa: E402
import torch  # noqa: E402

print("package:", os.path.dirname(H.__file__))
for g in sys.argv[2:]:
    st, s = (int(v) for v in g.split(":"))
    a = H.gen_poisson27(s, s, s) if st == 27 else H.gen_poisson7(s, s, s)
    f = H.ilu0(a)
    dp = H.DevicePrecond.create(a.n_rows, H.prepare_lower(f.l), H.prepare_upper(f.u))
    b = torch.tensor(H.spmv_csr(a, np.ones(a.n_rows)), device="cuda")
    x = torch.empty_like(b)
    for _ in range(3):
        dp.apply(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(10):
        e0.record()
        dp.apply(b, x)
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(f"{st}-pt {s}^3 ILU apply {np.median(ms):.4f} ms", flush=True)
