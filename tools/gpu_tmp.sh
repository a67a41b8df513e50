timeout 600 python tools/diag_fb_margin.py 4000 > gpurun_out/diag_fb.log 2>&1
timeout 900 python -m pytest tests/test_gpu_filterbank.py -q -rf -s > gpurun_out/pytest_fb.log 2>&1; echo "exit $?" >> gpurun_out/pytest_fb.log
