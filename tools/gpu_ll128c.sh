# LL128 after fusing the gather into the reduction loop: parity (loopback + 2 GPUs) and sweep.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -k "ll128 or back_to_back or bits_identical or check_ratios" > gpurun_out/pytest_ll128_loop.log 2>&1; echo "loopback exit $?"; tail -3 gpurun_out/pytest_ll128_loop.log
[ "$NG" -ge 2 ] && { timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "ll128 or variants or mixed" > gpurun_out/pytest_ll128_multi.log 2>&1; echo "multi exit $?"; tail -3 gpurun_out/pytest_ll128_multi.log; }
for dt in f32 bf16; do
timeout 900 $TR --master-port 29611 tools/k3_sweep.py --dtype $dt --variants 0,ll,ll128,push --sizes-mb 0.5,1,2,4,8,16,32,64 > gpurun_out/k3_ll128c_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
grep '^{' gpurun_out/k3_ll128c_${dt}_n${NG}.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('$dt', d['variant'], d['bucket_MB'], d['ours_ms'], d['ours_busbw'], d['nccl_busbw'])"
done
CANNIKIN_AR_LL128=1 CANNIKIN_AR_LL=0 timeout 600 $TR --master-port 29620 tools/k3_trace.py --sizes=4,16,64 > gpurun_out/k3_trace_ll128c_n${NG}.jsonl 2>/dev/null; echo "trace exit $?"
grep '^{' gpurun_out/k3_trace_ll128c_n${NG}.jsonl
