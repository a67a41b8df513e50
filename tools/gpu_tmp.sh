timeout 1500 python -m pytest tests -m gpu -q -rf --durations=8 > gpurun_out/pytest_r2a.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r2a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2a.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_r2a.log
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench exit $?" >> gpurun_out/bench_r2a.err
