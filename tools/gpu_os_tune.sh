export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29553 tools/k3_sweep.py --grids 4,8,9,10,12,16,32 --variants 0 --total 16777216 --sizes-mb 0.0625,0.25,0.5,1,2,4 > gpurun_out/k3_grid_small_n${NG}.jsonl 2>gpurun_out/k3_os_tune.err; echo "sweep exit $?"
python - <<PY
import json
rows=[json.loads(l) for l in open("gpurun_out/k3_grid_small_n${NG}.jsonl") if l.startswith("{")]
for r in rows: print(r["grid"], r["bucket_MB"], round(r["ours_ms"]*1e3/r["buckets"],2), "us/call")
PY
