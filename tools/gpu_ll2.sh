export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29661 tools/k3_sweep.py --variants 0,oneshot,ll --total 16777216 --sizes-mb 0.004,0.0625,0.25,0.5,1 > gpurun_out/k3_ll_n${NG}.jsonl 2>gpurun_out/k3_ll.err; echo "sweep exit $?"
timeout 600 $TR --master-port 29662 tools/k3_sweep.py --variants 0,ll --dtype bf16 --total 16777216 --sizes-mb 0.0625,0.5,1 > gpurun_out/k3_ll_bf16_n${NG}.jsonl 2>>gpurun_out/k3_ll.err; echo "sweep exit $?"
python - <<PY
import json
for f in ("gpurun_out/k3_ll_n${NG}.jsonl","gpurun_out/k3_ll_bf16_n${NG}.jsonl"):
  for l in open(f):
    if l.startswith("{"): r=json.loads(l); print(r["dtype"], r["variant"], r["bucket_MB"], round(r["ours_ms"]*1e3/r["buckets"],2), "us/call")
PY
grep -iE "error|trap" gpurun_out/k3_ll.err | head -3
