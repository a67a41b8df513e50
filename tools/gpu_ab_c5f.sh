#!/bin/bash
# C5 forward A/B of dev libraries (+ C5 forward parity tests on the last one)
TAG=$1; shift
mkdir -p gpurun_out
for v in "$@"; do SST_LIB_PATH=$PWD/paper_2003_07065_b200/$v NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5; done > gpurun_out/time_$TAG.log 2>&1
SST_LIB_PATH=$PWD/paper_2003_07065_b200/${@: -1} timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf -k "C5 or 12800 or nf512" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
