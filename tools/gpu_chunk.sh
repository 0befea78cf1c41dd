TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for c in 8192 4096 2048 1024; do
  export CANNIKIN_AR_CHUNK=$c
  echo "== chunk $c"
  timeout 300 $TR --master-port 29651 bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-hetero --no-nvls 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['value'], r['achieved'], r['kernel_ms'], r['kernel_ms_dist'])"
  timeout 300 $TR --master-port 29652 tools/k3_sweep.py --variants 1 --dtype bf16 --sizes-mb 64,256,1024 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'): r=json.loads(l); print(r['bucket_MB'], r['ours_busbw'])"
done
