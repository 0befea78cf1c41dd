export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_nvls.py -x -q > gpurun_out/pytest_nvls_n${NG}.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_nvls_n${NG}.log
timeout 600 $TR --master-port 29591 tools/k3_trace.py --nvls > gpurun_out/k6_trace_n${NG}.jsonl 2>gpurun_out/k6.err; echo "trace exit $?"
timeout 900 $TR --master-port 29581 tools/k3_sweep.py --dtype f32 --nvls --sizes-mb 4,16,64,256,1024 > gpurun_out/k6_sweep_n${NG}.jsonl 2>>gpurun_out/k6.err; echo "sweep exit $?"
grep '"rank": 0' gpurun_out/k6_trace_n${NG}.jsonl; cat gpurun_out/k6_sweep_n${NG}.jsonl; grep -E "Error" gpurun_out/k6.err | head -3
