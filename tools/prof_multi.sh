#!/bin/bash
# ncu --set full on forward+inverse of shortened C3 and C5 records (one launch each)
set -e
python tools/prof_run.py --cfg C3 --n-log2 20 > gpurun_out/prof_plain_c3.log 2>&1
python tools/prof_run.py --cfg C5 --n-log2 19 > gpurun_out/prof_plain_c5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel" -c 2 -o gpurun_out/prof_c3_$1 -f python tools/prof_run.py --cfg C3 --n-log2 20 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel" -c 2 -o gpurun_out/prof_c5_$1 -f python tools/prof_run.py --cfg C5 --n-log2 19 > gpurun_out/ncu_c5.log 2>&1
echo done
