#!/bin/bash
# One inverse iteration: narrow-band tests, C2/C3 timings (lib), ncu --set full of the C3 inverse.
#   gpurun -- 'bash tools/gpu_iter_inv.sh TAG [lib]'
TAG=${1:-it}; LIB=${2:-libsst.so}
mkdir -p gpurun_out
export SST_LIB_PATH=$PWD/paper_2003_07065_b200/$LIB
timeout 900 python -m pytest tests/test_gpu_inverse_nb.py tests/test_gpu_inverse.py -q -rf -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
if [ -n "$BOUNDS" ]; then SST_LIB_PATH=$PWD/paper_2003_07065_b200/libsst_bounds.so timeout 900 python -m pytest tests/test_gpu_inverse_nb.py -q -rf -x -k "isolated or subranges" > gpurun_out/pytest_bounds_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_bounds_$TAG.log; fi
for c in C2 C3; do timeout 300 python tools/time_cfg.py $c 10; done > gpurun_out/time_$TAG.log 2>&1
for v in $EXTRA; do SST_LIB_PATH=$PWD/paper_2003_07065_b200/$v timeout 300 python tools/time_cfg.py C3 10; done >> gpurun_out/time_$TAG.log 2>&1
python tools/prof_run.py --cfg C3 --n-log2 22 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"inv_" -c 1 \
    -o gpurun_out/prof_$TAG -f python tools/prof_run.py --cfg C3 --n-log2 22 > gpurun_out/ncu_$TAG.log 2>&1
echo done
