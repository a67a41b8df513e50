#!/bin/bash
# A/B of ridge DP builds: bash tools/gpu_ab_ridge.sh TAG lib...   (paper_2003_07065_b200/libsst_<lib>.so)
TAG=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab_ridge_$TAG.log
  for lam in 0.01 0; do SST_LIB_PATH=$PWD/paper_2003_07065_b200/libsst_$v.so timeout 120 python tools/ridge_prof.py $lam >> gpurun_out/ab_ridge_$TAG.log 2>&1; done
  SST_LIB_PATH=$PWD/paper_2003_07065_b200/libsst_$v.so timeout 300 python -m pytest tests/test_gpu_next.py -q -k "ridge" >> gpurun_out/ab_ridge_$TAG.log 2>&1
done
echo done
