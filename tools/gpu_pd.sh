export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k pushdyn > gpurun_out/pytest_pd_n${NG}.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_pd_n${NG}.log
timeout 900 $TR --master-port 29581 tools/k3_sweep.py --dtype f32 --variants 1,push,pushdyn:128,pushdyn:256,pushdyn:512,pushdyn:1024 --sizes-mb 16,64,256,1024 > gpurun_out/k3_pd_n${NG}.jsonl 2>gpurun_out/k3_pd.err; echo "sweep exit $?"
python - <<PY
import json
rows=[json.loads(l) for l in open("gpurun_out/k3_pd_n${NG}.jsonl") if l.startswith("{")]
for r in rows: print(r["variant"], r["bucket_MB"], r["ours_ms"], r["ours_busbw"], "nccl", r["nccl_busbw"])
PY
grep -iE "error|trap" gpurun_out/k3_pd.err | head -3
