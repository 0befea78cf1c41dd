# LL128 (flag-in-line two-shot) check: loopback tests on one GPU, multi-GPU parity, sweep vs the
# other variants at mid sizes.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -k "ll128 or back_to_back or bits_identical or check_ratios" > gpurun_out/pytest_ll128_loop.log 2>&1; echo "loopback exit $?"; tail -3 gpurun_out/pytest_ll128_loop.log
[ "$NG" -ge 2 ] && { timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "ll128 or variants or mixed" > gpurun_out/pytest_ll128_multi.log 2>&1; echo "multi exit $?"; tail -3 gpurun_out/pytest_ll128_multi.log; }
for dt in f32 bf16; do
[ "$NG" -ge 2 ] && timeout 900 $TR --master-port 29611 tools/k3_sweep.py --dtype $dt --variants 0,ll,ll128 --sizes-mb 0.25,1,2,4,8,16,32,64 > gpurun_out/k3_ll128_${dt}_n${NG}.jsonl 2>gpurun_out/k3_ll128_${dt}_n${NG}.err; echo "sweep $dt exit $?"
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/k3_ll128_*.jsonl")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f[-14:], d["variant"], d["bucket_MB"], d["ours_ms"], d["ours_busbw"], d["nccl_busbw"])
PY
