# A/B of the K2 kernel: build/ab/old.so vs build/ab/new.so, interleaved, same box.
L=paper_2402_05302_b200/libcannikin.so
for k in 1 2; do
for v in old new; do
cp build/ab/$v.so $L
timeout 600 python tools/k2_sweep.py --shapes c4,c4x2,c4f32,c5 --grids 0 --tma 0 --reps 10 2>/dev/null | grep '^{' | sed "s/^{/{\"build\": \"$v\", /" >> gpurun_out/k2_ab.jsonl
done
done
cp build/ab/new.so $L
python - <<'PY'
import json
for l in open("gpurun_out/k2_ab.jsonl"):
    d=json.loads(l); print(d["build"], d["shape"], d["variant"], d["grid"], d["ms"], d["GBps"])
PY
timeout 900 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/pytest_local.log 2>&1; echo "local tests exit $?"; tail -1 gpurun_out/pytest_local.log
