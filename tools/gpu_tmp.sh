timeout 300 python tools/time_cfg.py C3 1 > gpurun_out/plain_k.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"inv_kernel" -c 1 -o gpurun_out/prof_c3_inv_r2 python tools/time_cfg.py C3 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
