# 1-GPU: bench lines (graph), launch list, and one ncu --set full capture of the top kernel.
set -x
nvidia-smi -L
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c4.log 2>&1; echo "bench exit $?"
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_c1.log 2>&1; echo "bench c1 exit $?"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 300 $CMD --no-graph > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wsum_local -s 3 -c 1 -o gpurun_out/prof_k2_c4 $CMD --no-graph > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
tail -1 gpurun_out/bench_c4.log; tail -1 gpurun_out/bench_c1.log
