#!/bin/bash
# Round-2 GPU iteration: selected tests, a short bench per requested config.
#   TESTS="tests/test_gpu_shards.py ..."  CONFIGS="c2 c1"  BENCH_EXTRA="--no-cpu-baseline"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest $TESTS -m gpu -q -x -rs ${PYTEST_EXTRA} > gpurun_out/tests.txt 2>&1
  echo "TESTS_EXIT=$?" >> gpurun_out/tests.txt
  tail -5 gpurun_out/tests.txt
fi
for c in $CONFIGS; do
  timeout ${BENCH_TIMEOUT:-900} python bench.py --config $c --steps ${STEPS:-3} --warmup ${WARMUP:-3} $BENCH_EXTRA \
      > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?"; tail -c 600 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
