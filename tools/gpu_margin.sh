#!/bin/bash
# R23 margin experiment: GPU fp32 r error vs the model, then forward timings per margin factor.
TAG=${1:-m}
mkdir -p gpurun_out
timeout 900 python tools/diag_margin.py 2048 > gpurun_out/diag_margin_$TAG.log 2>&1
for M in 2 4 6 8; do
  SST_R23_M=$M timeout 300 python tools/time_cfg.py C3 5 | sed "s/^/M=$M /" >> gpurun_out/time_$TAG.log 2>&1
  SST_R23_M=$M NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 | sed "s/^/M=$M /" >> gpurun_out/time_$TAG.log 2>&1
done
SST_NO_REDECIDE=1 timeout 300 python tools/time_cfg.py C3 5 | sed 's/^/off /' >> gpurun_out/time_$TAG.log 2>&1
SST_NO_REDECIDE=1 NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 | sed 's/^/off /' >> gpurun_out/time_$TAG.log 2>&1
echo done
