timeout 900 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/pytest_local.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_local.log
timeout 900 python tools/k2_sweep.py --shapes c4q,c4h,c4,c4x2,c5bf16,c5,c3,c2,c1-big --grids 0 --altu-grids 0 > gpurun_out/k2_sweep4.jsonl 2> gpurun_out/k2_sweep4.err; echo "sweep exit $?"
cat gpurun_out/k2_sweep4.jsonl; tail -3 gpurun_out/k2_sweep4.err
