export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all_n${NG}.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_all_n${NG}.log
timeout 600 $TR --master-port 29531 tools/adaptive_batch.py > gpurun_out/adaptive_n${NG}.jsonl 2>gpurun_out/adaptive.err; echo "adaptive exit $?"
cat gpurun_out/adaptive_n${NG}.jsonl; tail -3 gpurun_out/adaptive.err
