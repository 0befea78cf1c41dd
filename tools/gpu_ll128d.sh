# (historical: CANNIKIN_LL128_FUSE existed only for this experiment and was removed after it)
# LL128 scatter fused into the reduction loop (CANNIKIN_LL128_FUSE=1) vs separate scatter phase.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
CANNIKIN_LL128_FUSE=1 timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -k "ll128 or back_to_back" > gpurun_out/pytest_ll128f_loop.log 2>&1; echo "loopback exit $?"; tail -1 gpurun_out/pytest_ll128f_loop.log
[ "$NG" -ge 2 ] && { CANNIKIN_LL128_FUSE=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "ll128 or variants" > gpurun_out/pytest_ll128f_multi.log 2>&1; echo "multi exit $?"; tail -1 gpurun_out/pytest_ll128f_multi.log; }
for f in 0 1; do
CANNIKIN_LL128_FUSE=$f timeout 900 $TR --master-port 2963$f tools/k3_sweep.py --dtype f32 --variants ll128 --sizes-mb 1,2,4,8,16,32,64 > gpurun_out/k3_ll128_fuse${f}_n${NG}.jsonl 2>/dev/null; echo "sweep fuse=$f exit $?"
grep '^{' gpurun_out/k3_ll128_fuse${f}_n${NG}.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('fuse $f', d['bucket_MB'], d['ours_ms'], d['ours_busbw'])"
done
CANNIKIN_LL128_FUSE=1 CANNIKIN_AR_LL128=1 CANNIKIN_AR_LL=0 timeout 600 $TR --master-port 29620 tools/k3_trace.py --sizes=4,16,64 > gpurun_out/k3_trace_ll128f_n${NG}.jsonl 2>/dev/null; echo "trace exit $?"
grep '^{' gpurun_out/k3_trace_ll128f_n${NG}.jsonl | cut -c1-250
