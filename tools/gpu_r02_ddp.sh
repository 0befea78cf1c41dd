#!/bin/bash
# Real ResNet-50/224 under torch DDP with the Cannikin comm hook, ranks capped by green contexts
# (tools/ddp_step.py --hetero sm): gated entry (full grid) vs round 1's ungated 24-CTA grid, W = 2, 4.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for W in 4 2; do
  DEV=$([ $W = 2 ] && echo 0,1 || echo 0,1,2,3)
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 $TR --nproc-per-node $W --master-port 2973$W tools/ddp_step.py --model resnet50 --img 224 --B $((128 * W)) --hetero sm > gpurun_out/ddp_step_sm_r50_n${W}_gated.jsonl 2>&1; echo "gated W=$W $?"
  CUDA_VISIBLE_DEVICES=$DEV timeout 900 $TR --nproc-per-node $W --master-port 2974$W tools/ddp_step.py --model resnet50 --img 224 --B $((128 * W)) --hetero sm --ungated --grid 24 > gpurun_out/ddp_step_sm_r50_n${W}_ungated24.jsonl 2>&1; echo "ungated24 W=$W $?"
done
grep -h summary gpurun_out/ddp_step_sm_r50_n*_*.jsonl
