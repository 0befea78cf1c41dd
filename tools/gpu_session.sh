#!/bin/bash
# One gpurun session, stages chosen by argument (run from the repo root on the GPU box):
#   tools/gpu_session.sh tests smoke bench launches ncu_k2 multi
#     tests     every -m gpu test (1..N GPUs)             -> gpurun_out/pytest_gpu_n<N>.log
#     smoke     __graft_entry__.smoke()                    -> gpurun_out/smoke.log
#     launches  ncu launch list of smoke (the driver's)    -> gpurun_out/launches_smoke.csv
#     bench     default bench line, and --bucket-mb 25     -> gpurun_out/bench_*.jsonl
#     ncu_k2    ncu --set full of the bench's K2 launch    -> gpurun_out/ncu_k2.ncu-rep
#     bench_multi  bench at N = all GPUs (torchrun)        -> gpurun_out/bench_n<N>.jsonl
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
    *) echo "unknown stage $stage" ;;
  esac
done
