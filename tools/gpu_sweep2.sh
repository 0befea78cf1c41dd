# C5 11-size bucket sweep (automatic variant) on the visible GPUs.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
for dt in f32 bf16; do
timeout 900 $TR --master-port 29603 tools/k3_sweep.py --dtype $dt --variants auto --sizes-mb 1,2,4,8,16,32,64,128,256,512,1024 > gpurun_out/k3_c5sweep_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
grep '^{' gpurun_out/k3_c5sweep_${dt}_n${NG}.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('$dt', d['bucket_MB'], d['ours_busbw'], d['nccl_busbw'], d['speedup_vs_nccl'])"
done
