export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
SZ=1,2,4,8,16,32,64,128,256,512,1024
for dt in f32 bf16; do
timeout 900 $TR --master-port 29603 tools/k3_sweep.py --dtype $dt --variants auto --sizes-mb $SZ > gpurun_out/k3_c5sweep_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
done
python - <<PY
import json
for dt in ("f32","bf16"):
  print(dt, [(r["bucket_MB"], r["ours_busbw"], r["speedup_vs_nccl"]) for r in (json.loads(l) for l in open(f"gpurun_out/k3_c5sweep_{dt}_n${NG}.jsonl") if l.startswith("{"))][:5])
PY
