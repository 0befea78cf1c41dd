export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_n${NG}.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_multi_n${NG}.log
timeout 900 $TR --master-port 29611 tools/k3_sweep.py --dtype bf16 --sizes-mb 4,16,64,256,1024 --variants 0,1,push > gpurun_out/k3_push_n${NG}.jsonl 2>gpurun_out/push.err; echo "sweep exit $?"
cat gpurun_out/k3_push_n${NG}.jsonl; grep -E "Error" gpurun_out/push.err | head -3
