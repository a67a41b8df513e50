#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench line, per-config timings, ncu launch list.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench exit $?" >> gpurun_out/bench_$TAG.err
for c in C2 C3 C4; do timeout 300 python tools/time_cfg.py $c 5 >> gpurun_out/time_$TAG.log 2>&1; done
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 >> gpurun_out/time_$TAG.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-traffic --legs none > gpurun_out/bench_short_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras --no-traffic --legs none \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_launch_$TAG.log
echo done
