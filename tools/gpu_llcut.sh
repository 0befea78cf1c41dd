# After lowering the LL limit to 1 MiB/(W-1): multi-GPU tests of the automatic path and LL, and the
# small/mid bucket sweep under the automatic choice.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_loopback.py -x -q -k "ll or mixed or variants or back_to_back" > gpurun_out/pytest_llcut_n${NG}.log 2>&1; echo "tests exit $?"; tail -1 gpurun_out/pytest_llcut_n${NG}.log
timeout 900 $TR --master-port 29681 tools/k3_sweep.py --dtype f32 --variants auto --total 16777216 --sizes-mb 0.25,0.5,0.75,1,1.5,2,4 2>/dev/null | grep '^{' > gpurun_out/k3_llcut_f32_n${NG}.jsonl; echo "sweep exit $?"
python - <<PY
import json
for l in open("gpurun_out/k3_llcut_f32_n${NG}.jsonl"):
    d=json.loads(l); print(d["bucket_MB"], round(d["ours_ms"]*1e3/d["buckets"],2), "us", d["ours_busbw"])
PY
