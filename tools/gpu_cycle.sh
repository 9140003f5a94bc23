#!/bin/bash
# Standard GPU iteration: gpu tests, a short bench, and the per-launch list of one bench step.
# Every step runs under its own timeout so a hang cannot hold the box.
export BENCH_NO_CLOCKS=1
timeout ${TEST_TIMEOUT:-400} python -m pytest tests -m "gpu ${TEST_FILTER}" -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/plain.log 2>&1 && tail -1 gpurun_out/plain.log | cut -c1-1100
if [ -z "$NO_NCU" ]; then
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu.log 2>&1
fi
