#!/bin/bash
# One gpurun call: GPU parity tests, smoke, default bench, ncu launch list + full
# captures of k_wave for the bench configs.
# usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh <tag>'
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $OUT/gpu.txt 2>&1
lscpu | head -20 > $OUT/lscpu.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-secondary --cpu-budget 0.1 > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 2 -c 1 \
    -o $OUT/wave_c2 python tools/one_solve.py --stencil 27 --size 128 --reps 3 > $OUT/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 2 -c 1 \
    -o $OUT/wave_c4 python tools/one_solve.py --stencil 7 --size 256 --reps 3 > $OUT/ncu_c4.log 2>&1
ls -la $OUT
