#!/bin/bash
# ncu --set full of one forward, its list-mode R23 repair launch and one inverse launch of the bench command (after a plain run);
# the report is summarised on the box (gpurun_out/ must stay under 64 MiB) and then deleted
TAG=${1:-r1}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras --no-traffic --legs none"
$CMD > gpurun_out/ncu_bench_plain_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel|inv_nb_kernel" -s 6 -c 3 \
   -o /tmp/prof_bench_$TAG -f $CMD > gpurun_out/ncu_bench_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench_$TAG.log
REP=/tmp/prof_bench_$TAG.ncu-rep
if [ -f $REP ]; then
  python tools/ncu_summary.py $REP > gpurun_out/ncu_summary_$TAG.txt 2>&1
  ncu -i $REP --page source --csv --print-source sass -k regex:fwd_kernel > /tmp/f.csv 2>/dev/null
  ncu -i $REP --page source --csv --print-source sass -k regex:"inv_kernel|inv_nb_kernel" > /tmp/i.csv 2>/dev/null
  python tools/ncu_sass.py /tmp/f.csv 6 > gpurun_out/ncu_sass_fwd_$TAG.txt 2>&1
  python tools/ncu_sass.py /tmp/i.csv 6 > gpurun_out/ncu_sass_inv_$TAG.txt 2>&1
  python tools/ncu_traffic.py $REP C3 1048576 gpurun_out/traffic_$TAG.json > /dev/null 2>&1
  rm -f $REP /tmp/f.csv /tmp/i.csv
fi
