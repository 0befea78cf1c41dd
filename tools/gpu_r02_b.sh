#!/bin/bash
# Round-2 session B (2 GPUs): the DDP-hook tests (world 1 and 2, oracle comparison), and the
# step-vs-DDP comparison with the gated entry at reduction grids 148 / 48 / 24.
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo buildfail; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_ddp.py -x -q > gpurun_out/pytest_ddp_n${NG}.log 2>&1; echo "ddp tests $?"; tail -2 gpurun_out/pytest_ddp_n${NG}.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $NG"
: > gpurun_out/hetero_grid_ab_n${NG}.jsonl
for grid in 0 48 24; do
  timeout 600 $TR --master-port $((29570 + grid)) bench.py --gpus $NG --no-nvls --no-e2e --hetero-grid $grid 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); h=d['step_vs_ddp']; print(json.dumps({'grid': $grid, **{k: h.get(k) for k in ['cannikin_ms','ddp_ms','saving','prediction_error','b_cannikin','learned_ms_per_sample','reduction']}}))" >> gpurun_out/hetero_grid_ab_n${NG}.jsonl
done
cat gpurun_out/hetero_grid_ab_n${NG}.jsonl
