set -x
timeout 900 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/pytest_local.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/pytest_local.log
timeout 900 python tools/k2_sweep.py > gpurun_out/k2_sweep.jsonl 2>gpurun_out/k2_sweep.err; echo "sweep exit $?"
cat gpurun_out/k2_sweep.jsonl; tail -5 gpurun_out/k2_sweep.err
