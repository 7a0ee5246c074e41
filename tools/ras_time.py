"""RAS GMRES time on one GPU (diagnostics): python tools/ras_time.py <package parent> [size]"""
import os
import sys
import time

sys.path.insert(0, os.path.abspath(sys.argv[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_00541_b200 as H  # noqa: E402
from paper_1606_00541_b200 import ras  # noqa: E402

s = int(sys.argv[2]) if len(sys.argv) > 2 else 64
a = H.gen_poisson7(s, s, s)
solver = ras.RasSolver(a, overlap=1, comm="none")
b = torch.tensor(H.spmv_csr(a, np.ones(a.n_rows)), device="cuda")
x = torch.zeros_like(b)
for k in range(int(os.environ.get("RAS_REPS", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = solver.gmres_device(b, x, restart=30)
    torch.cuda.synchronize()
    print(os.path.dirname(H.__file__), s, rep.iterations, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
