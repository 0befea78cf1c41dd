# 1-GPU round check: full GPU test suite, smoke, bench lines, launch list, ncu --set full of K2.
set -x
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench exit $?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 300 $CMD --no-graph > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wsum_local -s 3 -c 1 -o gpurun_out/prof_k2_c4_v2 $CMD --no-graph > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; tail -1 gpurun_out/bench_default.log
