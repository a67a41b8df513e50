NLIM=33554432 timeout 300 python tools/time_cfg.py C4 1 > gpurun_out/plain_k.log 2>&1 && \
NLIM=33554432 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c4.csv python tools/time_cfg.py C4 1 > gpurun_out/ncu_c4.log 2>&1
NLIM=16777216 timeout 300 python tools/time_cfg.py C5 3 > gpurun_out/time_c45.log 2>&1
timeout 300 python tools/time_cfg.py C3 3 >> gpurun_out/time_c45.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "C4 or C5 or C3 or C1" > gpurun_out/pytest_q.log 2>&1; echo "exit $?" >> gpurun_out/pytest_q.log
