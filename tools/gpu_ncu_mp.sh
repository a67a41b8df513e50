#!/bin/bash
# ncu --set full of the multi-pass (N_f = 2^15) kernels: one forward + one inverse of the §5.2
# Fig. 16(c) shape; summarised on the box, report deleted (gpurun_out/ must stay under 64 MiB)
TAG=${1:-r1}
mkdir -p gpurun_out
CMD="python tools/s52_timing.py --once"
$CMD > gpurun_out/ncu_mp_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mp_" \
   -o /tmp/prof_mp_$TAG -f $CMD > gpurun_out/ncu_mp_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_mp_$TAG.log
REP=/tmp/prof_mp_$TAG.ncu-rep
if [ -f $REP ]; then
  python tools/ncu_summary.py $REP > gpurun_out/ncu_summary_mp_$TAG.txt 2>&1
  rm -f $REP
fi
