#!/bin/bash
# One gpurun call: GPU parity tests, smoke, default bench (+ reference arm), ncu
# launch list of the bench, full captures of the dominant kernels.
# usage (from this container): gpurun --timeout 3000 -- 'bash tools/gpu_round.sh <tag>'
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
lscpu | head -20 > $OUT/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 600 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --secondary "" --ras-size 64 --ras-ref-size 0 --cpu-budget 0.1 \
    > $OUT/ncu_launch_bench.log 2>&1
for cfg in "27 128 L c2" "7 256 L c4" "7 256 U c4u"; do
    set -- $cfg
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 2 -c 1 \
        -o $OUT/wave_$4 python tools/one_solve.py --stencil $1 --size $2 --which $3 --reps 3 > $OUT/ncu_$4.log 2>&1
    ncu -i $OUT/wave_$4.ncu-rep --page raw --csv > $OUT/wave_$4_raw.csv 2>/dev/null
    ncu -i $OUT/wave_$4.ncu-rep --page source --csv --print-source sass > $OUT/wave_$4_source.csv 2>/dev/null
done
timeout 600 ncu --set full --clock-control none -k regex:k_spmv_hec -c 1 -o $OUT/spmv_c4 \
    python -c "
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1606_00541_b200 as H
a = H.gen_poisson7(256, 256, 256); s = H.DeviceSpmv(a); s.run_host(np.ones(a.n_cols))
" > $OUT/ncu_spmv.log 2>&1
ncu -i $OUT/spmv_c4.ncu-rep --page raw --csv > $OUT/spmv_c4_raw.csv 2>/dev/null
ls -la $OUT
