#!/bin/bash
# timings + GPU tests + one ncu --set full capture (C3 slice): bash tools/gpu_full.sh TAG
TAG=${1:-it}
mkdir -p gpurun_out
for c in C2 C3 C4; do timeout 300 python tools/time_cfg.py $c 5 >> gpurun_out/time_$TAG.log 2>&1; done
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 >> gpurun_out/time_$TAG.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
python tools/prof_run.py --cfg C3 --n-log2 21 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel|inv_nb_kernel" -c 2 \
    -o gpurun_out/prof_c3_$TAG -f python tools/prof_run.py --cfg C3 --n-log2 21 > gpurun_out/ncu_c3_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c3_$TAG.log
echo done
