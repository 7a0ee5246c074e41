#!/bin/bash
# Quick GPU iteration: parity tests + traces + strategy timing.
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python tools/trace_pipeline.py --stencil 27 --size 128 > $OUT/trace27.txt 2>&1
timeout 300 python tools/trace_pipeline.py --stencil 7 --size 256 > $OUT/trace7.txt 2>&1
timeout 600 python tools/devbench.py --grid 7:256 --grid 27:128 --ctas 148 --reps 10 --strategies 2 > $OUT/devbench.txt 2>&1
