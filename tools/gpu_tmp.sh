for M in 6; do
SST_R23_M=$M timeout 300 python tools/time_cfg.py C3 1 > gpurun_out/plain_k.log 2>&1 && \
SST_R23_M=$M timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_M$M.csv python tools/time_cfg.py C3 1 > gpurun_out/ncu_k.log 2>&1
done
SST_NO_REDECIDE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_off.csv python tools/time_cfg.py C3 1 > gpurun_out/ncu_k2.log 2>&1
echo done
