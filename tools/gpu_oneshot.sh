export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all_n${NG}.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_all_n${NG}.log
timeout 600 $TR --master-port 29551 tools/k3_sweep.py --variants 0,oneshot --total 16777216 --sizes-mb 0.004,0.0625,0.25,0.5,1,2,4 > gpurun_out/k3_oneshot_n${NG}.jsonl 2>gpurun_out/k3_oneshot.err; echo "sweep exit $?"
cat gpurun_out/k3_oneshot_n${NG}.jsonl | cut -c1-200; grep -iE "error|Trap" gpurun_out/k3_oneshot.err | head -5
