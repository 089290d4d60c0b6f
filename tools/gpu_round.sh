#!/bin/bash
# One gpurun call: GPU parity tests, the default bench line, the ncu launch
# list of a short bench run and one `ncu --set full` capture of the top SpMV
# kernel.  Usage (from this container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tests] [bench] [ncu] [full]'
set -u
mkdir -p gpurun_out
STAGES="${*:-tests bench ncu full}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/nproc.txt
for s in $STAGES; do
  case $s in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
      echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json ;;
    ref)
      timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1
      echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_ref.json ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --variants grid \
        --no-cpu-baseline --no-kdl --apps > gpurun_out/ncu_launch_bench.log 2>&1
      echo "ncu-launches rc=$?" ;;
    full)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:plan8_drain \
        -s 2 -c 1 -f -o gpurun_out/prof_spmv_grid python tools/prof_spmv.py grid --reps 3 \
        > gpurun_out/ncu_full.log 2>&1
      echo "ncu-full rc=$?"; tail -3 gpurun_out/ncu_full.log ;;
    appsncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_apps.csv python tools/prof_grid_apps.py 2 > gpurun_out/ncu_apps.log 2>&1
      for k in grid_persistent1 async_persistent; do
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -f \
          -o gpurun_out/prof_$k python tools/prof_grid_apps.py 2 >> gpurun_out/ncu_apps.log 2>&1
      done
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree.*grid_persistent" -s 1 -c 1 -f \
          -o gpurun_out/prof_tree_grid python tools/prof_grid_apps.py 2 >> gpurun_out/ncu_apps.log 2>&1
      echo "appsncu rc=$?"; tail -3 gpurun_out/ncu_apps.log ;;
    compare)
      timeout 900 ncu --replay-mode app-range --csv --log-file gpurun_out/compare_ncu.csv \
        --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,dram__sectors_read.sum,dram__sectors_write.sum \
        python tools/compare_metrics.py collect > gpurun_out/compare.log 2>&1
      timeout 600 python tools/compare_metrics.py report gpurun_out/compare_ncu.csv gpurun_out/compare.md >> gpurun_out/compare.log 2>&1
      echo "compare rc=$?"; tail -20 gpurun_out/compare.log ;;
    apps)
      timeout 1200 python tools/prof_apps.py --json gpurun_out/apps.json > gpurun_out/apps.log 2>&1
      echo "apps rc=$?"; tail -c 2000 gpurun_out/apps.log ;;
  esac
done
