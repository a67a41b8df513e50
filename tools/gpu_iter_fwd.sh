#!/bin/bash
# One forward iteration: forward parity tests, C2-C4 timings with and without the decision pre-test,
# ncu --set full of the C3 forward.   gpurun -- 'bash tools/gpu_iter_fwd.sh TAG [pytest -k expr]'
TAG=${1:-f}; KEXPR=${2:-}
mkdir -p gpurun_out
if [ -n "$KEXPR" ]; then K="-k $KEXPR"; else K=""; fi
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf -x $K > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
for c in C2 C3; do timeout 300 python tools/time_cfg.py $c 10; done > gpurun_out/time_$TAG.log 2>&1
NLIM=33554432 timeout 300 python tools/time_cfg.py C4 5 >> gpurun_out/time_$TAG.log 2>&1
for c in C2 C3; do SST_NO_PRETEST=1 timeout 300 python tools/time_cfg.py $c 10 | sed 's/^/no-pretest /'; done >> gpurun_out/time_$TAG.log 2>&1
SST_NO_PRETEST=1 NLIM=33554432 timeout 300 python tools/time_cfg.py C4 5 | sed 's/^/no-pretest /' >> gpurun_out/time_$TAG.log 2>&1
if [ -n "$PROF" ]; then
python tools/prof_run.py --cfg C3 --n-log2 22 --no-inverse > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel" -c 1 \
    -o gpurun_out/prof_$TAG -f python tools/prof_run.py --cfg C3 --n-log2 22 --no-inverse > gpurun_out/ncu_$TAG.log 2>&1
fi
echo done
