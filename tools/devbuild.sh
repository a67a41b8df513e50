#!/bin/bash
# Fast single-size build for register/spill inspection: tools/devbuild.sh 32 [extra nvcc flags]
N2=${1:-32}; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -cudart static -Xptxas -v -DSST_DEV_N2=$N2 "$@" -o ${OUT:-/tmp/libsst_dev.so} \
  paper_2003_07065_b200/csrc/sst_api.cu paper_2003_07065_b200/csrc/sst_kernels.cu paper_2003_07065_b200/csrc/ridge.cu paper_2003_07065_b200/csrc/multipass.cu 2>&1 | \
  grep -E "Compiling entry|registers|spill|error" | paste - - - | \
  sed -E "s/ptxas info *: Compiling entry function '_ZN3sst//; s/' for 'sm_100a'//; s/ptxas info *: Function properties for [^ ]*//; s/ptxas info *://" | cut -c1-200
