#!/bin/bash
# One forward iteration: forward-path GPU tests, C2-C5 timings, optional ncu of the C3 forward.
#   gpurun -- 'bash tools/gpu_iter_fwd.sh TAG'      (PROF=1: ncu --set full of the C3 forward)
TAG=${1:-f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_filterbank.py tests/test_gpu_dist.py tests/test_gpu_next.py -q -rf > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
for c in C2 C3; do timeout 300 python tools/time_cfg.py $c 10; done > gpurun_out/time_$TAG.log 2>&1
NLIM=33554432 timeout 300 python tools/time_cfg.py C4 5 >> gpurun_out/time_$TAG.log 2>&1
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 >> gpurun_out/time_$TAG.log 2>&1
if [ -n "$PROF" ]; then
python tools/prof_run.py --cfg C3 --n-log2 22 --no-inverse > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel" -c 1 \
    -o gpurun_out/prof_$TAG -f python tools/prof_run.py --cfg C3 --n-log2 22 --no-inverse > gpurun_out/ncu_$TAG.log 2>&1
fi
echo done
