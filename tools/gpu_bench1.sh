timeout 600 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/pytest_local.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_local.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c4.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --config c5 --steps 20 --warmup 5 --no-e2e > gpurun_out/bench_c5.log 2>&1; echo "bench c5 exit $?"
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo "bench c1 exit $?"
tail -1 gpurun_out/bench_c4.log; tail -1 gpurun_out/bench_c5.log; tail -1 gpurun_out/bench_c1.log
