#!/bin/bash
# ncu --set full of forward+inverse on a config slice: bash tools/gpu_prof_cfg.sh TAG CFG NLOG2
TAG=$1; CFG=$2; NL=$3
mkdir -p gpurun_out
python tools/prof_run.py --cfg $CFG --n-log2 $NL > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel|inv_nb_kernel" -c 2 \
    -o gpurun_out/prof_$TAG -f python tools/prof_run.py --cfg $CFG --n-log2 $NL > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$TAG.log
