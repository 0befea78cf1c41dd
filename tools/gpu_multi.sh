# 2+ GPU checks: multi-rank parity tests, the N-GPU bench (torchrun) and the K3-vs-NCCL sweep.
set -x
nvidia-smi -L
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_n${NG}.log 2>&1; echo "pytest multi exit $?"
timeout 600 $TR --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 > gpurun_out/bench_c4_n${NG}.log 2>&1; echo "bench n$NG exit $?"
timeout 600 $TR --master-port 29512 bench.py --gpus $NG --config c5 --steps 10 --warmup 3 --no-e2e > gpurun_out/bench_c5_n${NG}.log 2>&1; echo "bench c5 n$NG exit $?"
timeout 900 $TR --master-port 29513 tools/k3_sweep.py --dtype f32 --grids 64,148 > gpurun_out/k3_sweep_f32_n${NG}.jsonl 2>gpurun_out/k3_sweep_f32_n${NG}.err; echo "sweep f32 exit $?"
timeout 900 $TR --master-port 29514 tools/k3_sweep.py --dtype bf16 --grids 148 > gpurun_out/k3_sweep_bf16_n${NG}.jsonl 2>gpurun_out/k3_sweep_bf16_n${NG}.err; echo "sweep bf16 exit $?"
tail -3 gpurun_out/pytest_multi_n${NG}.log; tail -1 gpurun_out/bench_c4_n${NG}.log; tail -1 gpurun_out/bench_c5_n${NG}.log
cat gpurun_out/k3_sweep_f32_n${NG}.jsonl gpurun_out/k3_sweep_bf16_n${NG}.jsonl; tail -3 gpurun_out/k3_sweep_f32_n${NG}.err
