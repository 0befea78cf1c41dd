export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_n${NG}.log 2>&1; echo "pytest multi exit $?"; tail -2 gpurun_out/pytest_multi_n${NG}.log
for DT in bf16 f32; do
timeout 900 $TR --master-port 2951${#DT} tools/k3_sweep.py --dtype $DT --sizes-mb 16,64,256,1024 --variants 512:0,512:1,256:0,256:1 > gpurun_out/k3_tune_${DT}_n${NG}.jsonl 2>gpurun_out/k3_tune.err; echo "tune $DT exit $?"
done
cat gpurun_out/k3_tune_*_n${NG}.jsonl; tail -3 gpurun_out/k3_tune.err
