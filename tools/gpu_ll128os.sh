# One-shot LL128: parity (loopback + every visible GPU) and sweep vs LL / two-shot LL128 / two-shot.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -k "ll128 or back_to_back or bits_identical or check_ratios" > gpurun_out/pytest_ll128os_loop.log 2>&1; echo "loopback exit $?"; tail -1 gpurun_out/pytest_ll128os_loop.log
[ "$NG" -ge 2 ] && { timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "ll128os or variants" > gpurun_out/pytest_ll128os_multi_n${NG}.log 2>&1; echo "multi exit $?"; tail -1 gpurun_out/pytest_ll128os_multi_n${NG}.log; }
for dt in f32 bf16; do
timeout 900 $TR --master-port 29651 tools/k3_sweep.py --dtype $dt --variants ll,ll128os,ll128 --sizes-mb 0.0625,0.25,0.5,1,2,4,8,16 > gpurun_out/k3_ll128os_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
grep '^{' gpurun_out/k3_ll128os_${dt}_n${NG}.jsonl | python -c "
import sys,json
rows=[json.loads(l) for l in sys.stdin]
for r in rows: print('$dt', r['variant'], r['bucket_MB'], round(r['ours_ms']*1e3/r['buckets'],2), 'us', r['ours_busbw'])"
done
