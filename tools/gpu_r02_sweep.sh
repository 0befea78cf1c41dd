#!/bin/bash
# Round-2 refresh of the NVLink evidence on the final build (4-GPU box): the 11-size C5 bucket
# sweep (auto variant vs NCCL allreduce) at W = 4 and W = 2, f32 and bf16, and the N = 4 bench
# line with the live all-to-all ceiling.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo buildfail; exit 1; }
SZ=1,2,4,8,16,32,64,128,256,512,1024
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for dt in f32 bf16; do
  timeout 900 $TR --nproc-per-node 4 --master-port 2963$([ $dt = f32 ] && echo 1 || echo 2) tools/k3_sweep.py --dtype $dt --sizes-mb $SZ --variants auto > gpurun_out/k3_c5sweep_${dt}_n4.jsonl 2>&1; echo "sweep $dt n4 $?"
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 2964$([ $dt = f32 ] && echo 1 || echo 2) tools/k3_sweep.py --dtype $dt --sizes-mb $SZ --variants auto > gpurun_out/k3_c5sweep_${dt}_n2.jsonl 2>&1; echo "sweep $dt n2 $?"
done
timeout 900 $TR --nproc-per-node 4 --master-port 29651 bench.py --gpus 4 > gpurun_out/bench_n4_final.jsonl 2> gpurun_out/bench_n4_final.err; echo "bench n4 $?"
