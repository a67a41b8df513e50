timeout 300 python tools/ridge_prof.py 0.01 > gpurun_out/plain_r.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ridge_dp -c 1 -o gpurun_out/prof_ridge python tools/ridge_prof.py 0.01 > gpurun_out/ncu_r.log 2>&1
