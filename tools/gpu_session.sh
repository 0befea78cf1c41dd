#!/bin/bash
# One gpurun session, stages chosen by argument (run from the repo root on the GPU box):
#   tools/gpu_session.sh tests smoke bench launches ncu_k2 multi
#     tests     every -m gpu test (1..N GPUs)             -> gpurun_out/pytest_gpu_n<N>.log
#     smoke     __graft_entry__.smoke()                    -> gpurun_out/smoke.log
#     launches  ncu launch list of smoke (the driver's)    -> gpurun_out/launches_smoke.csv
#     bench     default bench line, and --bucket-mb 25     -> gpurun_out/bench_*.jsonl
#     ncu_k2    ncu --set full of the bench's K2 launch    -> gpurun_out/ncu_k2.ncu-rep
#     bench_multi  bench at N = all GPUs (torchrun)        -> gpurun_out/bench_n<N>.jsonl
#     nvls_bf16 the bf16 NVLS characterisation probe       -> gpurun_out/nvls_bf16_n<N>.jsonl
#     configs   every BASELINE config at N = 1, 2, 4       -> gpurun_out/configs_matrix.jsonl
#     sweep     11-size C5 bucket sweep, f32/bf16, W=N, 2  -> gpurun_out/k3_c5sweep_*.jsonl
#     ddp       ResNet-50 DDP hook, SM caps, gated vs 24   -> gpurun_out/ddp_step_sm_r50_*.jsonl
#     k2_ab / k3_ab  A/B of builds in build/variants/*.so  -> gpurun_out/k2_ab.jsonl, k3_ab.jsonl
#     stress    80k random-size calls per W, bit-exact       -> gpurun_out/stress.jsonl
set -u
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
echo "GPUs: $NG"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -20 gpurun_out/build.log; exit 1; }
for stage in "$@"; do
  case $stage in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_n${NG}.log 2>&1
      echo "tests exit $?"; tail -3 gpurun_out/pytest_gpu_n${NG}.log ;;
    tests_*)
      k=${stage#tests_}
      timeout 1500 python -m pytest tests -m gpu -x -q -k "$k" > gpurun_out/pytest_${k}_n${NG}.log 2>&1
      echo "tests[$k] exit $?"; tail -3 gpurun_out/pytest_${k}_n${NG}.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke exit $?"; tail -2 gpurun_out/smoke.log ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
        > gpurun_out/launches_smoke.log 2>&1
      echo "ncu launches exit $?"; tail -2 gpurun_out/launches_smoke.log
      grep -c gpu__time_duration gpurun_out/launches_smoke.csv ;;
    bench)
      timeout 600 python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err
      echo "bench exit $?"; tail -1 gpurun_out/bench_default.jsonl | cut -c1-400
      timeout 600 python bench.py --bucket-mb 25 > gpurun_out/bench_b25.jsonl 2> gpurun_out/bench_b25.err
      echo "bench b25 exit $?"; tail -1 gpurun_out/bench_b25.jsonl | cut -c1-400 ;;
    launches_bench)
      timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_plain.log 2>&1 &&
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu \
        > gpurun_out/launches_bench.log 2>&1
      echo "ncu bench launches exit $?" ;;
    ncu_k2)
      timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_plain2.log 2>&1 &&
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:wsum_local -s 3 -c 1 \
        -o gpurun_out/ncu_k2 -f python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_k2.log 2>&1
      echo "ncu k2 exit $?" ;;
    bench_multi)
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
        --master-port 29533 bench.py --gpus $NG > gpurun_out/bench_n${NG}.jsonl 2> gpurun_out/bench_n${NG}.err
      echo "bench n$NG exit $?"; tail -1 gpurun_out/bench_n${NG}.jsonl | cut -c1-600 ;;
    nvls_bf16)
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 \
        --master-port 29552 tools/nvls_bf16_probe.py > gpurun_out/nvls_bf16_n${NG}.jsonl 2>&1
      echo "nvls bf16 exit $?" ;;
    configs)
      : > gpurun_out/configs_matrix.jsonl
      for cfg in c1 c2 c3 c4 c5; do
        CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config $cfg --no-hetero --no-e2e --no-cpu \
          2>/dev/null | grep '^{' >> gpurun_out/configs_matrix.jsonl
        for W in 2 4; do
          [ "$NG" -ge $W ] || continue
          CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((W - 1))) timeout 600 python -m torch.distributed.run --nnodes=1 \
            --nproc-per-node $W --master-addr 127.0.0.1 --master-port $((29710 + W)) bench.py --gpus $W \
            --config $cfg --no-hetero --no-e2e --no-nvls 2>/dev/null | grep '^{' >> gpurun_out/configs_matrix.jsonl
        done
      done
      echo "configs: $(wc -l < gpurun_out/configs_matrix.jsonl) lines" ;;
    sweep)
      for dt in f32 bf16; do for W in $NG 2; do
        CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((W - 1))) timeout 900 python -m torch.distributed.run --nnodes=1 \
          --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29630 tools/k3_sweep.py --dtype $dt \
          --sizes-mb 1,2,4,8,16,32,64,128,256,512,1024 --variants auto > gpurun_out/k3_c5sweep_${dt}_n${W}.jsonl 2>&1
        echo "sweep $dt W=$W exit $?"
      done; done ;;
    ddp)
      for W in $NG 2; do
        for mode in gated ungated24; do
          extra=$([ $mode = gated ] && echo "" || echo "--ungated --grid 24")
          CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((W - 1))) timeout 900 python -m torch.distributed.run --nnodes=1 \
            --nproc-per-node $W --master-addr 127.0.0.1 --master-port 29735 tools/ddp_step.py --model resnet50 \
            --img 224 --B $((128 * W)) --hetero sm $extra > gpurun_out/ddp_step_sm_r50_n${W}_${mode}.jsonl 2>&1
          echo "ddp W=$W $mode exit $?"
        done
      done ;;
    k2_ab)
      : > gpurun_out/k2_ab.jsonl
      for rep in 1 2 3; do for lib in build/variants/*.so; do
        CANNIKIN_LIB=$PWD/$lib timeout 300 python tools/k2_vs_pattern.py --sets synth --k2-grids 0 \
          --pattern-grids 592 --tag $(basename $lib .so) 2>/dev/null | grep '^{' >> gpurun_out/k2_ab.jsonl
      done; done ;;
    k3_ab)
      : > gpurun_out/k3_ab.jsonl
      for rep in 1 2 3; do for lib in build/variants/*.so; do
        CANNIKIN_LIB=$PWD/$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG \
          --master-addr 127.0.0.1 --master-port $((29700 + rep)) bench.py --gpus $NG --no-hetero --no-e2e \
          --no-nvls --steps 30 2>/dev/null | grep '^{' | sed "s/^{/{\"lib\": \"$(basename $lib .so)\", /" \
          >> gpurun_out/k3_ab.jsonl
      done; done ;;
    stress)
      : > gpurun_out/stress.jsonl
      for W in 2 $NG; do for v in auto ll ll128 twoshot; do
        ME=$([ $v = ll ] && echo 131072 || echo 4194304)
        CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((W - 1))) timeout 900 python -m torch.distributed.run --nnodes=1 \
          --master-addr 127.0.0.1 --nproc-per-node $W --master-port $((29800 + W)) tools/stress_allreduce.py \
          --calls 10000 --variant $v --max-elems $ME 2>&1 | grep '^{' >> gpurun_out/stress.jsonl
      done; done; cat gpurun_out/stress.jsonl ;;
    *) echo "unknown stage $stage" ;;
  esac
done
