# 4-GPU round check after the LL128 variant: every GPU test, bench lines, auto-variant sweeps,
# DDP step (25 MB buckets now through LL128).
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all_${NG}gpu.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_all_${NG}gpu.log
bash tools/gpu_refresh.sh
timeout 900 $TR --master-port 29591 tools/ddp_step.py --model resnet50 --img 224 --B 512 --iters 8 --hetero sm > gpurun_out/ddp_step_sm_r50_n${NG}.jsonl 2>gpurun_out/ddp_sm.err; echo "ddp exit $?"; tail -1 gpurun_out/ddp_step_sm_r50_n${NG}.jsonl | cut -c1-600
