export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -k "ll or variant" > gpurun_out/pytest_ll_n${NG}.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_ll_n${NG}.log
timeout 600 $TR --master-port 29661 tools/k3_sweep.py --variants 0,oneshot,ll --total 16777216 --sizes-mb 0.004,0.0625,0.125,0.25 > gpurun_out/k3_ll_n${NG}.jsonl 2>gpurun_out/k3_ll.err; echo "sweep exit $?"
python - <<PY
import json
for l in open("gpurun_out/k3_ll_n${NG}.jsonl"):
    if l.startswith("{"): r=json.loads(l); print(r["variant"], r["bucket_MB"], round(r["ours_ms"]*1e3/r["buckets"],2), "us/call")
PY
grep -iE "error|trap" gpurun_out/k3_ll.err | head -3
