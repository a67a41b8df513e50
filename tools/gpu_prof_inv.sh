#!/bin/bash
# ncu --set full of the inverse kernels on a config slice for the given library:
#   bash tools/gpu_prof_inv.sh TAG CFG NLOG2 LIB [kernel regex]
TAG=$1; CFG=$2; NL=$3; LIB=$4; KR=${5:-inv_}
mkdir -p gpurun_out
export SST_LIB_PATH=$PWD/paper_2003_07065_b200/$LIB
python tools/prof_run.py --cfg $CFG --n-log2 $NL > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -c 1 \
    -o gpurun_out/prof_$TAG -f python tools/prof_run.py --cfg $CFG --n-log2 $NL > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$TAG.log
