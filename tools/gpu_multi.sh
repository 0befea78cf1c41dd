# 2+ GPU checks: multi-rank parity tests, then the N-GPU bench (torchrun) and the DDP baseline.
set -x
nvidia-smi -L; nvidia-smi topo -m | head -5
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi.log 2>&1; echo "pytest multi exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 > gpurun_out/bench_n${NG}.log 2>&1; echo "bench n$NG exit $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $NG --config c5 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_c5_n${NG}.log 2>&1; echo "bench c5 n$NG exit $?"
tail -15 gpurun_out/pytest_multi.log; tail -1 gpurun_out/bench_n${NG}.log; tail -1 gpurun_out/bench_c5_n${NG}.log
