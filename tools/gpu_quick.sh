#!/bin/bash
# One gpurun call for a build-measure iteration: GPU tests (all, no -x), then C2-C5 timings with and
# without the R23 re-decision.   gpurun --timeout 1800 -- 'bash tools/gpu_quick.sh TAG [pytest args]'
TAG=${1:-q}
shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 "$@" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
for c in C2 C3 C4; do timeout 300 python tools/time_cfg.py $c 5 >> gpurun_out/time_$TAG.log 2>&1; done
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 >> gpurun_out/time_$TAG.log 2>&1
for c in C3; do SST_NO_REDECIDE=1 timeout 300 python tools/time_cfg.py $c 5 | sed 's/^/no-redecide /' >> gpurun_out/time_$TAG.log 2>&1; done
SST_NO_REDECIDE=1 NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 | sed 's/^/no-redecide /' >> gpurun_out/time_$TAG.log 2>&1
echo done
