NLIM=16777216 timeout 300 python tools/time_cfg.py C5 5 > gpurun_out/time_c5.log 2>&1
timeout 300 python tools/time_cfg.py C3 5 >> gpurun_out/time_c5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "C5 or nf512 or nf128 or nf256 or extreme or degenerate" > gpurun_out/pytest_c5.log 2>&1; echo "exit $?" >> gpurun_out/pytest_c5.log
