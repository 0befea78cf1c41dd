# Refresh the bench lines and the C5 bucket sweep on this box (all visible GPUs, and N = 1).
export CANNIKIN_SPIN_TIMEOUT_MS=15000
NG=$(nvidia-smi -L | wc -l)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
SZ=1,2,4,8,16,32,64,128,256,512,1024
[ "$NG" -gt 2 ] && CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_c4_n1.log 2>&1; echo "bench n1 exit $?"; tail -1 gpurun_out/bench_c4_n1.log | cut -c1-300
timeout 600 $TR --master-port 29601 bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4_n${NG}.log 2>&1; echo "bench c4 exit $?"; tail -1 gpurun_out/bench_c4_n${NG}.log | cut -c1-300
timeout 600 $TR --master-port 29602 bench.py --config c5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5_n${NG}.log 2>&1; echo "bench c5 exit $?"; tail -1 gpurun_out/bench_c5_n${NG}.log | cut -c1-300
for dt in f32 bf16; do
timeout 900 $TR --master-port 29603 tools/k3_sweep.py --dtype $dt --variants auto --sizes-mb $SZ > gpurun_out/k3_c5sweep_${dt}_n${NG}.jsonl 2>/dev/null; echo "sweep $dt exit $?"
done
