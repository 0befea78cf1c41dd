export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
for h in 0 2 1; do
  if [ $h = 0 ]; then python -m paper_2402_05302_b200.build -f > /dev/null; else CANNIKIN_NVCC_EXTRA="-DCANNIKIN_LD_HINT=$h" python -m paper_2402_05302_b200.build > /dev/null; fi
  CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/k2_sweep.py --shapes c4,c5,c4x3 --grids 0 --tma 0 > gpurun_out/k2_ldhint$h.jsonl 2>/dev/null; echo "k2 hint $h exit $?"
  timeout 600 $TR --master-port 2961$h tools/k3_sweep.py --variants 0,1 --sizes-mb 16,64,256 > gpurun_out/k3_ldhint$h.jsonl 2>/dev/null; echo "k3 hint $h exit $?"
done
python -m paper_2402_05302_b200.build -f > /dev/null
for h in 0 2 1; do python - $h <<'PY'
import json,sys
h=sys.argv[1]
for l in open(f"gpurun_out/k2_ldhint{h}.jsonl"):
    if l.startswith("{"): r=json.loads(l); print("K2 hint",h, {k:r[k] for k in r if k in ("shape","variant","grid","dyn","us","GBps","gbps","ms")})
for l in open(f"gpurun_out/k3_ldhint{h}.jsonl"):
    if l.startswith("{"): r=json.loads(l); print("K3 hint",h, r["variant"], r["bucket_MB"], r["ours_busbw"])
PY
done
