# A/B of LL128 builds (build/ab/*.so) on the visible GPUs, interleaved.
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
L=paper_2402_05302_b200/libcannikin.so
cp $L /tmp/keep.so
for k in 1 2; do
for v in u2 u4 g4; do
cp build/ab/$v.so $L
CANNIKIN_SPIN_TIMEOUT_MS=15000 timeout 600 $TR --master-port 2967$k tools/k3_sweep.py --dtype f32 --variants ll128 --sizes-mb 1,2,4,8,16 2>/dev/null | grep '^{' | sed "s/^{/{\"build\": \"$v\", /" >> gpurun_out/ll128_ab.jsonl
done
done
cp /tmp/keep.so $L
python - <<'PY'
import json, collections
d=collections.defaultdict(list)
for l in open("gpurun_out/ll128_ab.jsonl"):
    r=json.loads(l); d[(r["bucket_MB"], r["build"])].append(r["ours_busbw"])
for k in sorted(d): print(k, d[k])
PY
