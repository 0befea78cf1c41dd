# Final 2-GPU check: every GPU test, the C4 and C5 bench lines at N = 2.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all_${NG}gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_all_${NG}gpu.log
timeout 600 $TR --master-port 29601 bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4_n${NG}.log 2>&1; echo "bench c4 exit $?"; tail -1 gpurun_out/bench_c4_n${NG}.log | cut -c1-300
timeout 600 $TR --master-port 29602 bench.py --config c5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5_n${NG}.log 2>&1; echo "bench c5 exit $?"; tail -1 gpurun_out/bench_c5_n${NG}.log | cut -c1-300
