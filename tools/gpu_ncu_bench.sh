#!/bin/bash
# ncu --set full of one forward and one inverse launch of the bench command (after a plain run)
TAG=${1:-r1}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extras"
$CMD > gpurun_out/ncu_bench_plain_$TAG.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|inv_kernel" -s 6 -c 2 \
   -o gpurun_out/prof_bench_$TAG -f $CMD > gpurun_out/ncu_bench_$TAG.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench_$TAG.log
