export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_full.py -x -q > gpurun_out/pytest_multi_n${NG}.log 2>&1; echo "pytest multi exit $?"; tail -2 gpurun_out/pytest_multi_n${NG}.log
timeout 600 $TR --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 > gpurun_out/bench_c4_n${NG}.log 2>&1; echo "bench n$NG exit $?"
tail -1 gpurun_out/bench_c4_n${NG}.log; grep -i -E "error|Traceback" gpurun_out/bench_c4_n${NG}.log | head
