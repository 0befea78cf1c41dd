export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_bw tools/nvlink_bw.cu
for g in 148 296; do timeout 60 tools/nvlink_bw 256 $g 512; done > gpurun_out/nvlink_bw_n${NG}.jsonl 2>&1; grep a2a gpurun_out/nvlink_bw_n${NG}.jsonl
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_nvls.py -x -q > gpurun_out/pytest_multi_n${NG}.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_multi_n${NG}.log
timeout 600 $TR --master-port 29561 bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4_n${NG}.log 2>&1; echo "bench exit $?"; tail -1 gpurun_out/bench_c4_n${NG}.log | cut -c1-600
timeout 600 $TR --master-port 29562 tools/k3_sweep.py --variants auto --total 16777216 --sizes-mb 0.0625,0.25,0.5,1,2,4 > gpurun_out/k3_auto_small_n${NG}.jsonl 2>/dev/null; echo "sweep exit $?"
python - <<PY
import json
rows=[json.loads(l) for l in open("gpurun_out/k3_auto_small_n${NG}.jsonl") if l.startswith("{")]
for r in rows: print(r["variant"], r["bucket_MB"], round(r["ours_ms"]*1e3/r["buckets"],2), "us/call", "nccl", round(r["nccl_ms"]*1e3/r["buckets"],2))
PY
