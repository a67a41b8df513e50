#!/bin/bash
# Ridge DP iteration: f1 GPU tests + C1 ridge timings (tools/ridge_prof.py) for several lambda.
#   gpurun --timeout 900 -- 'bash tools/gpu_ridge.sh TAG'
TAG=${1:-ridge}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_next.py -q -rf -k "ridge or zone or mode" > gpurun_out/pytest_ridge_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_ridge_$TAG.log
for lam in 0.01 0.1 1e-4 0; do timeout 120 python tools/ridge_prof.py $lam >> gpurun_out/ridge_$TAG.log 2>&1; done
echo done
