set -x
nvidia-smi -L
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; echo "bench exit $?"
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo "bench c1 exit $?"
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench_c4.log
