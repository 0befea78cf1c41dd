#!/bin/bash
# N = 4 (and N = 2) bench lines with the live all-to-all ceiling probe (cannikin_probe_a2a_write).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29681 bench.py --gpus 4 --no-hetero --no-e2e --no-nvls 2>/dev/null | grep '^{' > gpurun_out/bench_n4_probe.jsonl; echo "bench4 $?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29682 bench.py --gpus 2 --no-hetero --no-e2e --no-nvls 2>/dev/null | grep '^{' > gpurun_out/bench_n2_probe.jsonl; echo "bench2 $?"
