# K4 fast path (fp32 PreMulSum): parity on every visible GPU and sweep.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "nccl or static" > gpurun_out/pytest_k4b_n${NG}.log 2>&1; echo "tests exit $?"; tail -1 gpurun_out/pytest_k4b_n${NG}.log
for dt in f32 bf16; do
timeout 900 $TR --master-port 29641 tools/k3_sweep.py --dtype $dt --variants auto,k4 --sizes-mb 1,4,16,64,256,1024 > gpurun_out/k4_sweep_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
grep '^{' gpurun_out/k4_sweep_${dt}_n${NG}.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('$dt', d['variant'], d['bucket_MB'], d['ours_busbw'], 'nccl-ar', d['nccl_busbw'])"
done
