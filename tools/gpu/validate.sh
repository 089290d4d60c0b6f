#!/bin/bash
# One GPU call: the GPU test suite, then a default bench run (outputs under gpurun_out/).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest.txt 2>&1
tail -5 gpurun_out/pytest.txt
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  head -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
fi
