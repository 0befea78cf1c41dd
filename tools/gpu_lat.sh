export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi_n${NG}.log 2>&1; echo "pytest multi exit $?"; tail -2 gpurun_out/pytest_multi_n${NG}.log
timeout 900 $TR --master-port 29515 tools/k3_sweep.py --dtype f32 --grids 148 --total 4194304 --sizes-mb 0.004,0.0625,0.25,1,4,16 > gpurun_out/k3_lat_n${NG}.jsonl 2>gpurun_out/k3_lat.err; echo "lat exit $?"
timeout 900 $TR --master-port 29516 tools/k3_sweep.py --dtype f32 --grids 148 > gpurun_out/k3_sweep_f32_n${NG}.jsonl 2>>gpurun_out/k3_lat.err; echo "sweep exit $?"
cat gpurun_out/k3_lat_n${NG}.jsonl gpurun_out/k3_sweep_f32_n${NG}.jsonl; tail -3 gpurun_out/k3_lat.err
