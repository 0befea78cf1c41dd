TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for v in "DYN=1 PUSH=0" "DYN=0 PUSH=0" "DYN=0 PUSH=1" "DYN=0 PUSH=2"; do
  eval "export CANNIKIN_AR_$(echo $v | cut -d' ' -f1) CANNIKIN_AR_$(echo $v | cut -d' ' -f2)"
  echo "== $v"
  timeout 300 $TR --master-port 29641 tools/k3_trace.py --bf16 --sizes=209.808 2>/dev/null | grep rank
done
