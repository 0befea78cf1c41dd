export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "pushdyn or oneshot" > gpurun_out/pytest_pd_n${NG}.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_pd_n${NG}.log
timeout 600 $TR --master-port 29553 tools/k3_sweep.py --variants 0,oneshot --total 16777216 --sizes-mb 0.0625,0.125,0.25,0.5,1,2 > gpurun_out/k3_os_n${NG}.jsonl 2>/dev/null; echo "sweep exit $?"
python - <<PY
import json
rows=[json.loads(l) for l in open("gpurun_out/k3_os_n${NG}.jsonl") if l.startswith("{")]
for r in rows: print(r["variant"], r["bucket_MB"], round(r["ours_ms"]*1e3/r["buckets"],2), "us/call")
PY
timeout 900 $TR --master-port 29581 tools/k3_sweep.py --dtype f32 --variants push,pushdyn:256,pushdyn:512 --sizes-mb 64,256,1024 > gpurun_out/k3_pd_n${NG}.jsonl 2>/dev/null; echo "sweep exit $?"
python - <<PY
import json
rows=[json.loads(l) for l in open("gpurun_out/k3_pd_n${NG}.jsonl") if l.startswith("{")]
for r in rows: print(r["variant"], r["bucket_MB"], r["ours_ms"], r["ours_busbw"], "nccl", r["nccl_busbw"])
PY
timeout 900 $TR --master-port 29591 tools/ddp_step.py --model resnet50 --img 224 --B 512 --iters 8 --hetero sm > gpurun_out/ddp_step_sm_r50_n${NG}.jsonl 2>gpurun_out/ddp_sm.err; echo "ddp exit $?"; tail -1 gpurun_out/ddp_step_sm_r50_n${NG}.jsonl
