SST_R23_M=6 timeout 300 python tools/time_cfg.py C3 1 > gpurun_out/plain_k.log 2>&1 && \
SST_R23_M=6 timeout 900 ncu --set full --import-source on --clock-control none -k regex:fwd_kernel -c 1 -o gpurun_out/prof_fwd_r23 python tools/time_cfg.py C3 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
