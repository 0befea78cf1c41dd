# A/B of K2 builds (build/ab/*.so), interleaved on one box.
L=paper_2402_05302_b200/libcannikin.so
cp $L /tmp/keep.so
for k in 1 2; do
for v in mb4 mb5 mb6; do
cp build/ab/$v.so $L
timeout 600 python tools/k2_sweep.py --shapes c4,c4f32,c5 --grids 0 --tma 0 --reps 10 2>/dev/null | grep '^{' | sed "s/^{/{\"build\": \"$v\", /" >> gpurun_out/k2_ab3.jsonl
done
done
cp /tmp/keep.so $L
python - <<'PY'
import json, collections
d=collections.defaultdict(list)
for l in open("gpurun_out/k2_ab3.jsonl"):
    r=json.loads(l); d[(r["shape"], r["build"])].append(r["ms"])
for k in sorted(d): print(k, sorted(d[k]))
PY
