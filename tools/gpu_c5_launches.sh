#!/bin/bash
# ncu launch list (gpu__time_duration) of the C5 forward sequence + inverse on a 2^22-sample slice,
# and ncu --set full of the redecide kernel and the full-band inverse (summaries only).
TAG=${1:-r2}
mkdir -p gpurun_out
python tools/prof_run.py --cfg C5 --n-log2 22 > gpurun_out/prof_plain_c5l_$TAG.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$TAG.csv \
    python tools/prof_run.py --cfg C5 --n-log2 22 > gpurun_out/ncu_c5l_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c5l_$TAG.log
timeout 900 ncu --set full --clock-control none -k regex:"redecide_kernel|inv_nb_kernel|inv_kernel" -c 2 \
    -o /tmp/prof_c5b_$TAG -f python tools/prof_run.py --cfg C5 --n-log2 22 > gpurun_out/ncu_c5b_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c5b_$TAG.log
[ -f /tmp/prof_c5b_$TAG.ncu-rep ] && python tools/ncu_summary.py /tmp/prof_c5b_$TAG.ncu-rep > gpurun_out/ncu_summary_c5b_$TAG.txt 2>&1
rm -f /tmp/prof_c5b_$TAG.ncu-rep
echo done
