#!/bin/bash
# K3 A/B of library builds in build/variants/*.so on the N-GPU bench line (C4), interleaved.
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $NG"
: > gpurun_out/k3_ab.jsonl
for rep in 1 2 3; do for lib in build/variants/*.so; do
  tag=$(basename $lib .so)
  CANNIKIN_LIB=$PWD/$lib timeout 600 $TR --master-port $((29700 + rep)) bench.py --gpus $NG --no-hetero --no-e2e --no-nvls --steps 30 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); r=d['roofline']; print(json.dumps({'lib': '$tag', 'kernel_ms': r['kernel_ms'], 'busbw': r['achieved'], 'p50': r['kernel_ms_dist']['p50'], 'variant': r['kernel']}))" >> gpurun_out/k3_ab.jsonl
done; done
cat gpurun_out/k3_ab.jsonl
