#!/bin/bash
# Round-end evidence in one gpurun call: ncu --set full of the bench's C3 forward + inverse
# (gpu_ncu_bench.sh) and of the C5 forward + full-band inverse on a 2^22-sample slice; reports are
# summarised on the box and deleted (gpurun_out/ stays small).
#   gpurun --timeout 2400 -- 'bash tools/gpu_final.sh TAG'
TAG=${1:-r2}
mkdir -p gpurun_out
bash tools/gpu_ncu_bench.sh $TAG
python tools/prof_run.py --cfg C5 --n-log2 22 > gpurun_out/prof_plain_c5_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel|inv_nb_kernel" -c 2 \
    -o /tmp/prof_c5_$TAG -f python tools/prof_run.py --cfg C5 --n-log2 22 > gpurun_out/ncu_c5_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c5_$TAG.log
REP=/tmp/prof_c5_$TAG.ncu-rep
if [ -f $REP ]; then
  python tools/ncu_summary.py $REP > gpurun_out/ncu_summary_c5_$TAG.txt 2>&1
  ncu -i $REP --page source --csv --print-source sass -k regex:fwd_kernel > /tmp/f5.csv 2>/dev/null
  python tools/ncu_sass.py /tmp/f5.csv 6 > gpurun_out/ncu_sass_fwd_c5_$TAG.txt 2>&1
  rm -f $REP /tmp/f5.csv
fi
echo done
