#!/bin/bash
# A/B of the paired-tap fp64 re-decision (libsst_pair.so, -DSST_REDECIDE_PAIR=1) against libsst.so:
# C3/C5 timings, then the forward-path GPU tests on the variant.
TAG=${1:-pair}
mkdir -p gpurun_out
R=$PWD/paper_2003_07065_b200
for lib in libsst.so libsst_pair.so; do
  SST_LIB_PATH=$R/$lib timeout 300 python tools/time_cfg.py C3 10
  NLIM=16777216 SST_LIB_PATH=$R/$lib timeout 300 python tools/time_cfg.py C5 5
  NLIM=33554432 SST_LIB_PATH=$R/$lib timeout 300 python tools/time_cfg.py C4 5
done > gpurun_out/time_$TAG.log 2>&1
SST_LIB_PATH=$R/libsst_pair.so timeout 1300 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
cat gpurun_out/time_$TAG.log; tail -3 gpurun_out/pytest_$TAG.log
