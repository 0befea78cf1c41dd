#!/bin/bash
# Round-2 multi-GPU session (run from the repo root on a 2- or 4-GPU box): every -m gpu test, the
# bench at N = all GPUs (and N = 2 when there are 4), the bf16 NVLS characterisation probe.
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo buildfail; tail -30 gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_n${NG}.log 2>&1; echo "tests $?"; tail -3 gpurun_out/pytest_gpu_n${NG}.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node $NG --master-port 29551 bench.py --gpus $NG > gpurun_out/bench_n${NG}.jsonl 2> gpurun_out/bench_n${NG}.err; echo "bench n$NG $?"
timeout 600 $TR --nproc-per-node $NG --master-port 29552 tools/nvls_bf16_probe.py > gpurun_out/nvls_bf16_n${NG}.jsonl 2>&1; echo "nvls bf16 $?"
if [ "$NG" -ge 4 ]; then
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29553 bench.py --gpus 2 > gpurun_out/bench_n2.jsonl 2> gpurun_out/bench_n2.err; echo "bench n2 $?"
fi
