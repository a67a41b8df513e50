for i in 1 2; do timeout 300 python tools/time_cfg.py C3 5 >> gpurun_out/time_f.log 2>&1; done
NLIM=33554432 timeout 300 python tools/time_cfg.py C4 3 >> gpurun_out/time_f.log 2>&1
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 3 >> gpurun_out/time_f.log 2>&1
timeout 300 python tools/time_cfg.py C2 3 >> gpurun_out/time_f.log 2>&1
timeout 900 python -m pytest tests/test_gpu_inverse.py tests/test_gpu_parity.py -q -x -k "inverse" > gpurun_out/pytest_inv.log 2>&1; echo "exit $?" >> gpurun_out/pytest_inv.log
