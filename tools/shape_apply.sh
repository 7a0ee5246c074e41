# ILU apply time (b = A*1) per solver shape (G K RPL); default = planner's choice
cat > /tmp/sa.py <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1606_00541_b200 as H
grids = [g.split(":") for g in sys.argv[1:]]
for st, s in grids:
    st, s = int(st), int(s)
    a = H.gen_poisson27(s, s, s) if st == 27 else H.gen_poisson7(s, s, s)
    f = H.ilu0(a)
    try:
        dp = H.DevicePrecond.create(a.n_rows, H.prepare_lower(f.l), H.prepare_upper(f.u))
    except Exception as e:
        print(f"{os.environ.get('TAG','auto')} {st}-pt {s}^3: {e}"); continue
    b = torch.tensor(H.spmv_csr(a, np.ones(a.n_rows)), device="cuda")
    x = torch.empty_like(b)
    for _ in range(3): dp.apply(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(10):
        e0.record(); dp.apply(b, x); e1.record(); e1.synchronize(); ms.append(e0.elapsed_time(e1))
    print(f"{os.environ.get('TAG','auto')} {st}-pt {s}^3 ILU apply {np.median(ms):.4f} ms", flush=True)
PY
GRIDS="$@"
python /tmp/sa.py $GRIDS
for sh in "1 4 2" "2 4 2" "4 2 4" "8 2 2"; do set -- $sh; TAG="G=$1,K=$2,R=$3" HEC_WAVE_G=$1 HEC_WAVE_K=$2 HEC_WAVE_RPL=$3 python /tmp/sa.py $GRIDS; done
