#!/bin/bash
# quick iteration: per-config timings + GPU tests (+ optional extra command)
TAG=${1:-it}
mkdir -p gpurun_out
for c in C2 C3 C4; do timeout 300 python tools/time_cfg.py $c 5 >> gpurun_out/time_$TAG.log 2>&1; done
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 >> gpurun_out/time_$TAG.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
if [ -n "$2" ]; then eval "$2" > gpurun_out/extra_$TAG.log 2>&1; fi
echo done
