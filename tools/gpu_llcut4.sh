# Automatic-variant sweep 0.25-16 MB on the visible GPUs (after the LL128 grid change).
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29681 tools/k3_sweep.py --dtype f32 --variants auto --total 16777216 --sizes-mb 0.25,0.5,1,2,4,8,16 2>/dev/null | grep '^{' > gpurun_out/k3_gpw1_f32_n${NG}.jsonl; echo "sweep exit $?"
python - <<PY
import json
for l in open("gpurun_out/k3_gpw1_f32_n${NG}.jsonl"):
    d=json.loads(l); print(d["bucket_MB"], round(d["ours_ms"]*1e3/d["buckets"],2), "us", d["ours_busbw"])
PY
