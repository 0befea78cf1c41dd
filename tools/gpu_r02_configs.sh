#!/bin/bash
# Every BASELINE config at N = 1, 2, 4 (4-GPU box), bench line without the sidecars that do not
# depend on the config: one JSON line per (config, N) in gpurun_out/configs_matrix.jsonl.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
: > gpurun_out/configs_matrix.jsonl
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for cfg in c1 c2 c3 c4 c5; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config $cfg --no-hetero --no-e2e --no-cpu 2>/dev/null | grep '^{' >> gpurun_out/configs_matrix.jsonl; echo "$cfg n1 $?"
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29711 bench.py --gpus 2 --config $cfg --no-hetero --no-e2e --no-nvls 2>/dev/null | grep '^{' >> gpurun_out/configs_matrix.jsonl; echo "$cfg n2 $?"
  timeout 600 $TR --nproc-per-node 4 --master-port 29712 bench.py --gpus 4 --config $cfg --no-hetero --no-e2e --no-nvls 2>/dev/null | grep '^{' >> gpurun_out/configs_matrix.jsonl; echo "$cfg n4 $?"
done
