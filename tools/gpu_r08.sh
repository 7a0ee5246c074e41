mkdir -p gpurun_out/r08
timeout 600 python -m pytest tests/ -m gpu -x -q > gpurun_out/r08/pytest.log 2>&1
for r in 2 4 8; do echo "rpl=$r"; HEC_WAVE_RPL=$r timeout 300 python tools/devbench.py --grid 7:256 --grid 27:128 --grid 7:128 --ctas 148 --reps 10 --strategies 2 2>&1 | grep strat; done > gpurun_out/r08/rpl.txt 2>&1
HEC_WAVE_RPL=4 timeout 600 python -m pytest tests/test_gpu_trisolve.py -x -q > gpurun_out/r08/pytest_rpl4.log 2>&1
HEC_DEBUG=1 timeout 600 python - > gpurun_out/r08/rcm.txt 2>&1 <<'PY'
import sys, os; sys.path.insert(0, '.')
import numpy as np, paper_1606_00541_b200 as H
sys.path.insert(0, 'tools')
from config_sweep import timed_lu
for s in (100, 128):
    a = H.gen_poisson7(s, s, s)
    for name, perm in (("rcm", H.rcm_ordering(a)), ("random", H.random_ordering(a.n_rows, 1606))):
        ap = H.permute_symmetric(a, perm)
        b = H.spmv_csr(ap, np.ones(a.n_rows))
        f = H.ilu0(ap)
        ms, alg, info = timed_lu(H.prepare_lower(f.l), H.prepare_upper(f.u), b)
        print(s, name, round(ms, 3), "ms", round(alg / ms / 1e6, 1), "GB/s", flush=True)
PY
