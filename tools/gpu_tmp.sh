NLIM=33554432 timeout 300 python tools/time_cfg.py C4 3 > gpurun_out/time_c4.log 2>&1
NLIM=33554432 SST_NO_REDECIDE=1 timeout 300 python tools/time_cfg.py C4 3 >> gpurun_out/time_c4.log 2>&1
NLIM=33554432 timeout 300 python tools/time_cfg.py C4 1 > gpurun_out/plain_k.log 2>&1 && \
NLIM=33554432 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c4.csv python tools/time_cfg.py C4 1 > gpurun_out/ncu_c4.log 2>&1
