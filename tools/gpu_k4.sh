# K4 (NCCL path) check: parity on every visible GPU, sweep vs the P2P kernels and NCCL allreduce,
# bench line with the k4 sidecar.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "nccl" > gpurun_out/pytest_k4_n${NG}.log 2>&1; echo "k4 tests exit $?"; tail -2 gpurun_out/pytest_k4_n${NG}.log
for dt in f32 bf16; do
timeout 900 $TR --master-port 29641 tools/k3_sweep.py --dtype $dt --variants auto,k4 --sizes-mb 1,4,16,64,256,1024 > gpurun_out/k4_sweep_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
grep '^{' gpurun_out/k4_sweep_${dt}_n${NG}.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('$dt', d['variant'], d['bucket_MB'], d['ours_busbw'], 'nccl-ar', d['nccl_busbw'])"
done
timeout 600 $TR --master-port 29642 bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4_k4_n${NG}.log 2>&1; echo "bench exit $?"
tail -1 gpurun_out/bench_c4_k4_n${NG}.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ddp_baseline'])"
