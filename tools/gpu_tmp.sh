NLIM=16777216 timeout 300 python tools/time_cfg.py C5 3 > gpurun_out/plain_k.log 2>&1 && \
NLIM=16777216 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5b.csv python tools/time_cfg.py C5 1 > gpurun_out/ncu_k.log 2>&1
timeout 300 python tools/time_cfg.py C3 5 >> gpurun_out/plain_k.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or multipass" > gpurun_out/pytest_q.log 2>&1; echo "exit $?" >> gpurun_out/pytest_q.log
