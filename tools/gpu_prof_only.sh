#!/bin/bash
# one ncu --set full capture of the forward+inverse kernels on a C3 slice: bash tools/gpu_prof_only.sh TAG
TAG=${1:-p}
mkdir -p gpurun_out
python tools/prof_run.py --cfg C3 --n-log2 21 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel|inv_nb_kernel" -c 2 \
    -o gpurun_out/prof_c3_$TAG -f python tools/prof_run.py --cfg C3 --n-log2 21 > gpurun_out/ncu_c3_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c3_$TAG.log
