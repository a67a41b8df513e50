timeout 600 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/pytest_dist.log 2>&1; echo "exit $?" >> gpurun_out/pytest_dist.log
SST_LIB=bounds timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_bounds.log 2>&1; echo "exit $?" >> gpurun_out/pytest_bounds.log
