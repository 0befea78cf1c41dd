# 1-GPU: launch list + one ncu --set full capture of K2 in the bench command (current build).
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1; echo "plain exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 300 $CMD --no-graph > gpurun_out/plain2.log 2>&1; echo "plain2 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wsum_local -s 3 -c 1 -o gpurun_out/prof_k2_c4_r01b $CMD --no-graph > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
ls -la gpurun_out/prof_k2_c4_r01b.ncu-rep
