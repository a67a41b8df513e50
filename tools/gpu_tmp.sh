timeout 300 python tools/time_fb.py C2 > gpurun_out/plain_fb.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_fb.csv python tools/time_fb.py C2 > gpurun_out/ncu_fb.log 2>&1
