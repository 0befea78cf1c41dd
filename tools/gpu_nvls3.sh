export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_multi.py -q -x -k "nvls or push" > gpurun_out/pytest_nvls_push_n${NG}.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_nvls_push_n${NG}.log
timeout 900 $TR --master-port 29621 tools/k3_sweep.py --dtype f32 --variants auto --nvls --sizes-mb 16,64,256,1024 > gpurun_out/k6_vs_k3_n${NG}.jsonl 2>/dev/null; echo "sweep exit $?"
python - <<PY
import json
for l in open("gpurun_out/k6_vs_k3_n${NG}.jsonl"):
    if l.startswith("{"): r=json.loads(l); print(r["bucket_MB"], "K3", r["ours_busbw"], "K6", r["nvls_busbw"], "NCCL", r["nccl_busbw"])
PY
