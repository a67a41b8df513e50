#!/bin/bash
# Inverse-path iteration: narrow-band tests, then C2/C3 timings of the given dev libraries with the
# narrow-band path and with SST_INV_NB=0.   gpurun -- 'bash tools/gpu_ab_inv.sh TAG lib1 lib2 ...'
TAG=${1:-nb}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_inverse_nb.py tests/test_gpu_inverse.py -q -rf -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
for v in "$@"; do
  for c in C2 C3; do
    SST_LIB_PATH=$PWD/paper_2003_07065_b200/$v timeout 300 python tools/time_cfg.py $c 10
  done
done > gpurun_out/time_$TAG.log 2>&1
SST_INV_NB=0 timeout 300 python tools/time_cfg.py C3 10 | sed 's/^/residue-split /' >> gpurun_out/time_$TAG.log 2>&1
echo done
