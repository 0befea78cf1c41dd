# 4 GPUs after the LL128 range change: smoke, the auto-variant tests, DDP step, C5 auto sweep.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_ddp.py -x -q -k "mixed or ddp or ll128" > gpurun_out/pytest_auto_n${NG}.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_auto_n${NG}.log
timeout 900 $TR --master-port 29591 tools/ddp_step.py --model resnet50 --img 224 --B 512 --iters 8 --hetero sm > gpurun_out/ddp_step_sm_r50_n${NG}.jsonl 2>gpurun_out/ddp_sm.err; echo "ddp exit $?"; tail -1 gpurun_out/ddp_step_sm_r50_n${NG}.jsonl | cut -c1-700
for dt in f32 bf16; do
timeout 900 $TR --master-port 29603 tools/k3_sweep.py --dtype $dt --variants auto --sizes-mb 1,2,4,8,16,32,64,128,256,512,1024 > gpurun_out/k3_c5sweep_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
grep '^{' gpurun_out/k3_c5sweep_${dt}_n${NG}.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('$dt', d['bucket_MB'], d['ours_busbw'], d['nccl_busbw'], d['speedup_vs_nccl'])"
done
