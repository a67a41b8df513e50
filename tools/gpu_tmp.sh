mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-extras --legs '' > gpurun_out/bench_tr.log 2>&1; echo "exit $?" >> gpurun_out/bench_tr.log
