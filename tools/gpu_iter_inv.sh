#!/bin/bash
# One inverse iteration: narrow-band + inverse tests (and the bounds build with BOUNDS=1), C2/C3/C5
# timings, optional ncu (PROF=CFG) of the inverse.   gpurun -- 'bash tools/gpu_iter_inv.sh TAG'
TAG=${1:-it}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_inverse_nb.py tests/test_gpu_inverse.py -q -rf > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
if [ -n "$BOUNDS" ]; then SST_LIB=bounds timeout 900 python -m pytest tests/test_gpu_inverse_nb.py -q -rf -k "isolated or subranges" > gpurun_out/pytest_bounds_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_bounds_$TAG.log; fi
for c in C2 C3; do timeout 300 python tools/time_cfg.py $c 10; done > gpurun_out/time_$TAG.log 2>&1
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 >> gpurun_out/time_$TAG.log 2>&1
SST_INV_NB=0 NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 | sed 's/^/residue-split /' >> gpurun_out/time_$TAG.log 2>&1
if [ -n "$PROF" ]; then
python tools/prof_run.py --cfg $PROF --n-log2 22 > gpurun_out/prof_plain_$TAG.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"inv_" -c 1 \
    -o gpurun_out/prof_$TAG -f python tools/prof_run.py --cfg $PROF --n-log2 22 > gpurun_out/ncu_$TAG.log 2>&1
fi
echo done
