# (historical: CANNIKIN_LL128_MODE existed only for this experiment and was removed after it)
# LL128 experiments: store flavour / poll backoff (CANNIKIN_LL128_MODE) and a phase trace.
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
for m in 0 1 2 3; do
CANNIKIN_LL128_MODE=$m timeout 600 $TR --master-port 2961$m tools/k3_sweep.py --dtype f32 --variants ll128 --sizes-mb 4,16,64 > gpurun_out/k3_ll128_mode${m}_n${NG}.jsonl 2>/dev/null; echo "mode $m exit $?"
grep '^{' gpurun_out/k3_ll128_mode${m}_n${NG}.jsonl | python -c "
import sys,json
for l in sys.stdin: d=json.loads(l); print('mode $m', d['bucket_MB'], d['ours_ms'], d['ours_busbw'])"
done
CANNIKIN_AR_LL128=1 CANNIKIN_AR_LL=0 timeout 600 $TR --master-port 29620 tools/k3_trace.py --sizes=4,16,64 > gpurun_out/k3_trace_ll128_n${NG}.jsonl 2>/dev/null; echo "trace exit $?"
grep '^{' gpurun_out/k3_trace_ll128_n${NG}.jsonl
