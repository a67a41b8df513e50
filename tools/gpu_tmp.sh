timeout 900 python tools/time_fb.py C2 C3 C4 > gpurun_out/time_fb.log 2>&1
timeout 300 python tools/time_fb.py C2 > gpurun_out/plain_fb.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_fb.csv python tools/time_fb.py C2 > gpurun_out/ncu_fb.log 2>&1
timeout 900 python -m pytest tests/test_gpu_filterbank.py -q -rf > gpurun_out/pytest_fb.log 2>&1; echo "exit $?" >> gpurun_out/pytest_fb.log
